// SPDX-License-Identifier: Apache-2.0
//
// K3 — particle -> cell mapping (SubBlockRegistry::build + build_fraction_field,
//      psm.cpp:55-136); set_solid_velocities (psm.cpp:138-169) is evaluated inside the PSM
//      kernels from the snapshots (v_snap), setu_kernel only materialises the field
// K4 — hydrodynamic force/torque reduction (finalize_hydro_forces, psm.cpp:278-322)
//
// Mapping design (B200): the reference tests every particle against k^3 = 512 host
// sub-blocks and then every cell against its sub-block list (~67 candidates per cell in
// config 3). Here the particle list is binned on the device into 8^3-cell bins; each bin's
// candidate list is sorted ascending by snapshot index (= id order), so a cell sees a
// superset of the reference's eps > 0 candidates in the same order and the first-two /
// third-is-overfull rule (psm.cpp:103-130) gives identical entries. One thread per cell
// writes count/btot for every cell (coalesced, as the reference does) and, per entry, the
// id and B. The solid velocity u + omega x (c - x) of an entry is not stored: the PSM
// kernels compute it from the snapshot list current at sweep time (set_solid_velocities'
// post-sync list, sim.cpp:249-267 and 296-297), with the same operations as setu_kernel, so
// the 24 B per entry write (here) and read (K2) of v0/v1 are gone.
//
// Reduction design: PARITY mode reproduces the reference's per-particle Neumaier sums in
// lexicographic cell order bitwise: every fraction entry of the covered-cell lists becomes a
// (particle, cell, slot) key, a radix sort puts each particle's entries in the reference's
// visiting order, and six threads per particle run the compensated chains (f.x..t.z) over
// the particle's segment. FAST sums the same segments plainly; the fused force mode
// (lbg_sweep.cu) sums inside the PSM kernel with warp aggregation + atomics instead.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "lbg_internal.cuh"

namespace lbg {

constexpr int kBin = 8;  // bin edge in cells

struct BinGeom {
    int nb[3];
    int lo[3];    // block box lo (global cell coords)
    int dims[3];  // block dims
};

__device__ __forceinline__ bool bin_range(const BinGeom& g, const lbg_snapshot& p, int blo[3], int bhi[3]) {
    // cells whose reach-box test (psm.cpp:66-81: AABB distance <= r + 1/2) can pass
    const double reach = p.r + 0.5;
    for (int a = 0; a < 3; ++a) {
        const double lo = p.x[a] - reach - g.lo[a];
        const double hi = p.x[a] + reach - g.lo[a];
        int c0 = (int)floor(lo) - 1, c1 = (int)floor(hi) + 1;  // generous, the cell test is exact
        c0 = max(c0, 0);
        c1 = min(c1, g.dims[a] - 1);
        if (c1 < c0) return false;
        blo[a] = c0 / kBin;
        bhi[a] = c1 / kBin;
    }
    return true;
}

__global__ void bin_count_kernel(const lbg_snapshot* __restrict__ s, int n, BinGeom g, int* __restrict__ cnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int lo[3], hi[3];
    if (!bin_range(g, s[p], lo, hi)) return;
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) atomicAdd(&cnt[(z * g.nb[1] + y) * g.nb[0] + x], 1);
}

__global__ void bin_fill_kernel(const lbg_snapshot* __restrict__ s, int n, BinGeom g,
                                const int* __restrict__ start, int* __restrict__ cursor,
                                int* __restrict__ items) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int lo[3], hi[3];
    if (!bin_range(g, s[p], lo, hi)) return;
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                const int b = (z * g.nb[1] + y) * g.nb[0] + x;
                const int pos = atomicAdd(&cursor[b], 1);
                items[start[b] + pos] = p;
            }
}

// per-bin ascending order (= id order) makes the candidate sequence deterministic
__global__ void bin_sort_kernel(const int* __restrict__ start, const int* __restrict__ cnt, int nbins,
                                int* __restrict__ items) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbins) return;
    int* a = items + start[b];
    const int n = cnt[b];
    for (int i = 1; i < n; ++i) {
        const int v = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = v;
    }
}

struct MapArgs {
    const lbg_snapshot* __restrict__ s;
    BinGeom g;
    const int* __restrict__ start;
    const int* __restrict__ cnt;
    const int* __restrict__ items;
    uint8_t* __restrict__ count;
    int* __restrict__ id0;
    int* __restrict__ id1;
    double* __restrict__ b0;
    double* __restrict__ b1;
    double* __restrict__ btot;
    double* __restrict__ v0;
    double* __restrict__ v1;
    DeviceErrors* err;
    int* cov_n;
};

// K3 mapping (psm.cpp:28-32 overlap_fraction, psm.cpp:93-136 per-cell entry rule): one CTA
// per 8^3 bin, two cells per thread. The bin's candidate
// snapshots are staged in shared memory in list (= id) order, 64 at a time, so every lane reads
// the same candidate (broadcast) and the loop has no per-lane trip count. The overlap test is
// overlap_fraction (psm.cpp:28-32) with two exact shortcuts on the squared distance d2 =
// (dx*dx + dy*dy) + dz*dz (the radicand the reference takes the root of):
//   d2 > (r + f_r)^2 (1 + 1e-9)      => eps <= 0 (skip), the rounding of the root and of
//                                       -(dist - r) + f_r is ~1e-16 relative, far inside the
//                                       margin;
//   d2 < (r + f_r - 1)^2 (1 - 1e-9)  => eps >= 1, which the clamp makes exactly 1.0.
// Every other candidate takes the reference's sqrt path, so count/ids/fractions are bitwise
// those of build_fraction_field. Segment lists are registered
// by a separate pass (segments_kernel), since a warp here is not a row segment.
constexpr int kMapCand = 64;

// distance from x to the interval [lo, hi] of cell-centre coordinates, as |c - x| of its
// nearest member c is computed (c - x rounded; for x > hi, x - hi = -(hi - x) exactly)
__device__ __forceinline__ double axis_gap(double lo, double hi, double x) {
    return x < lo ? lo - x : (x > hi ? x - hi : 0.0);
}

__global__ void __launch_bounds__(256, 4) map_bin_kernel(const MapArgs a) {
    const BinGeom& g = a.g;
    const int b = blockIdx.x;
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    __shared__ double sx0[kMapCand], sx1[kMapCand], sx2[kMapCand], sr[kMapCand], sfr[kMapCand];
    __shared__ double sout2[kMapCand], sin2[kMapCand];
    __shared__ int sid[kMapCand];
    const int t = threadIdx.x;
    const int i = bx * kBin + (t & 7), j = by * kBin + ((t >> 3) & 7);
    int k[2] = {bz * kBin + (t >> 6), bz * kBin + (t >> 6) + 4};
    bool valid[2];
    long long c[2];
    double cc0 = (double)(g.lo[0] + i) + 0.5, cc1 = (double)(g.lo[1] + j) + 0.5, cc2[2];
    int cnt[2] = {0, 0};
    double sum[2] = {0.0, 0.0};
    bool over[2] = {false, false};
    for (int h = 0; h < 2; ++h) {
        valid[h] = i < g.dims[0] && j < g.dims[1] && k[h] < g.dims[2];
        c[h] = ((long long)k[h] * g.dims[1] + j) * g.dims[0] + i;
        cc2[h] = (double)(g.lo[2] + k[h]) + 0.5;
    }
    // cell-centre box of this warp's cells: x 8, y 4 (z per h)
    const int lane = t & 31;
    const int wj = by * kBin + (((t & ~31) >> 3) & 7);
    const double wx0 = (double)(g.lo[0] + bx * kBin) + 0.5, wx1 = (double)(g.lo[0] + bx * kBin + 7) + 0.5;
    const double wy0 = (double)(g.lo[1] + wj) + 0.5, wy1 = (double)(g.lo[1] + wj + 3) + 0.5;
    const int n = a.cnt[b];
    if (n == 0) return;  // count and btot of the whole field were zeroed before the launch
    const int* list = a.items + a.start[b];
    for (int base = 0; base < n; base += kMapCand) {
        const int m = min(kMapCand, n - base);
        __syncthreads();
        if (t < m) {
            const lbg_snapshot& p = a.s[list[base + t]];
            sx0[t] = p.x[0];
            sx1[t] = p.x[1];
            sx2[t] = p.x[2];
            sr[t] = p.r;
            sfr[t] = p.f_r;
            const double ro = p.r + p.f_r, ri = ro - 1.0;
            sout2[t] = (ro * ro) * (1.0 + 1e-9);
            sin2[t] = ri > 0.0 ? (ri * ri) * (1.0 - 1e-9) : -1.0;
            sid[t] = p.id;
        }
        __syncthreads();
        for (int h = 0; h < 2; ++h) {
            // warp-level cull: a candidate enters the cell loop only if it can reach a cell
            // centre of this warp's 8 x 4 x 1 row block. The squared gap between the candidate
            // and the box of cell centres bounds every cell's radicand from below in floating
            // point too (each per-axis gap is the smallest |c - x| over the box, and rounding
            // is monotonic), so the box rejects only candidates every cell rejects (rad > sout2)
            unsigned rel[2];
            for (int half = 0; half < 2; ++half) {
                const int q = lane + 32 * half;
                bool r = false;
                if (q < m) {
                    const double g0 = axis_gap(wx0, wx1, sx0[q]), g1 = axis_gap(wy0, wy1, sx1[q]);
                    const double g2 = axis_gap(cc2[h], cc2[h], sx2[q]);
                    r = !((g0 * g0 + g1 * g1) + g2 * g2 > sout2[q]);
                }
                rel[half] = __ballot_sync(0xffffffffu, r);
            }
            if (!valid[h] || over[h]) continue;
            for (int half = 0; half < 2 && !over[h]; ++half) {
                for (unsigned mask = rel[half]; mask; mask &= mask - 1) {  // ascending = id order
                    const int q = 32 * half + __ffs(mask) - 1;
                    const double d0 = cc0 - sx0[q], d1 = cc1 - sx1[q], d2 = cc2[h] - sx2[q];
                    const double rad = (d0 * d0 + d1 * d1) + d2 * d2;
                    if (rad > sout2[q]) continue;
                    double eps;
                    if (rad < sin2[q]) {
                        eps = 1.0;
                    } else {
                        eps = -(sqrt(rad) - sr[q]) + sfr[q];
                        eps = eps < 0.0 ? 0.0 : (1.0 < eps ? 1.0 : eps);  // std::clamp
                        if (eps <= 0.0) continue;
                    }
                    if (cnt[h] >= 2) {
                        over[h] = true;
                        break;
                    }
                    if (cnt[h] == 0) {
                        a.id0[c[h]] = sid[q];
                        a.b0[c[h]] = eps;
                    } else {
                        a.id1[c[h]] = sid[q];
                        a.b1[c[h]] = eps;
                    }
                    ++cnt[h];
                    sum[h] += eps;
                }
            }
        }
    }
    for (int h = 0; h < 2; ++h) {
        if (valid[h] && cnt[h] > 0) {  // uncovered cells keep the zeroed count and btot (+0.0)
            a.count[c[h]] = (uint8_t)cnt[h];
            a.btot[c[h]] = sum[h] < 1.0 ? sum[h] : 1.0;  // std::min(1.0, sum)
        }
        covered_count(valid[h] ? cnt[h] : 0, a.cov_n);
        const unsigned mo = __ballot_sync(0xffffffffu, over[h]);
        if (mo && (t & 31) == 0) atomicAdd(&a.err->overfull, (unsigned long long)__popc(mo));
    }
}

// the zero fills of one mapping in one launch (instead of six memsets, each an API call that
// the block-worker threads sharing a GPU serialise on): the bin counters and cursors, the
// scan's leading zero, the covered/segment counters, and count (u8) + btot (+0.0) of every
// cell — what build_fraction_field stores for an uncovered cell (psm.cpp:128-129). A thread
// clears 16 cells (one 16-byte count chunk, 128 bytes of btot).
__global__ void __launch_bounds__(256) map_zero_kernel(int* __restrict__ bins2, long long nbins2,
                                                       int* __restrict__ start0, int* __restrict__ cov_n,
                                                       int* __restrict__ seg_n, uint8_t* __restrict__ count,
                                                       double* __restrict__ btot, long long cells) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nbins2) bins2[t] = 0;
    if (t < 2) {
        cov_n[t] = 0;
        seg_n[t] = 0;
    }
    if (t == 0) *start0 = 0;
    const long long c0 = 16 * t;
    if (c0 + 16 <= cells) {
        reinterpret_cast<uint4*>(count)[t] = make_uint4(0u, 0u, 0u, 0u);
        double2* bt = reinterpret_cast<double2*>(btot + c0);
#pragma unroll
        for (int u = 0; u < 8; ++u) bt[u] = make_double2(0.0, 0.0);
    } else {
        for (long long c = c0; c < cells; ++c) {
            count[c] = 0;
            btot[c] = 0.0;
        }
    }
}

// covered-cell list from an externally set fraction field
__global__ void __launch_bounds__(256) covered_kernel(const uint8_t* __restrict__ count, long long cells,
                                                      int* __restrict__ n) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    covered_count(c < cells ? count[c] : 0, n);
}

// segment lists from an externally set fraction field (one thread per 32-cell row segment)
__global__ void __launch_bounds__(256) segments_kernel(const uint8_t* __restrict__ count, int nx, long long rows,
                                                       unsigned* __restrict__ seg_list, int* __restrict__ seg_n,
                                                       long long seg_cap) {
    const int per_row = (nx + 31) / 32;
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= rows * per_row) return;
    const long long row = s / per_row;
    const int i0 = (int)(s % per_row) * 32;
    const long long c0 = row * nx + i0;
    int mx = 0;
    for (int i = 0; i < 32 && i0 + i < nx; ++i) mx = max(mx, (int)count[c0 + i]);
    if (mx == 1)
        seg_list[atomicAdd(&seg_n[0], 1)] = (unsigned)c0;
    else if (mx >= 2)
        seg_list[seg_cap - 1 - atomicAdd(&seg_n[1], 1)] = (unsigned)c0;
}

// psm.cpp:138-169 — standalone setU over an existing fraction field
__global__ void __launch_bounds__(256) setu_kernel(const lbg_snapshot* __restrict__ s, SnapIndex sidx, BinGeom g,
                                                   const uint8_t* __restrict__ count,
                                                   const int* __restrict__ id0, const int* __restrict__ id1,
                                                   double* __restrict__ v0, double* __restrict__ v1,
                                                   DeviceErrors* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    int unknown = 0;
    if (i < g.dims[0]) {
        const long long c = ((long long)k * g.dims[1] + j) * g.dims[0] + i;
        const int cnt = count[c];
        const double cc[3] = {(double)(g.lo[0] + i) + 0.5, (double)(g.lo[1] + j) + 0.5,
                              (double)(g.lo[2] + k) + 0.5};
        for (int e = 0; e < cnt; ++e) {
            const int p = sidx(e == 0 ? id0[c] : id1[c]);
            if (p < 0) {
                ++unknown;
                continue;
            }
            const double r0 = cc[0] - s[p].x[0], r1 = cc[1] - s[p].x[1], r2 = cc[2] - s[p].x[2];
            const double* w = s[p].omega;
            double* v = (e == 0 ? v0 : v1) + 3 * c;
            v[0] = s[p].u[0] + (w[1] * r2 - w[2] * r1);
            v[1] = s[p].u[1] + (w[2] * r0 - w[0] * r2);
            v[2] = s[p].u[2] + (w[0] * r1 - w[1] * r0);
        }
    }
    unsigned v = unknown;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (v && (threadIdx.x & 31) == 0) atomicAdd(&err->unknown, (unsigned long long)v);
}

// ---------------------------------------------------------------- K4 reduction
__device__ __forceinline__ void nm_add(double& sum, double& comp, double v) {  // vec3.hpp:75-82
    const double t = sum + v;
    if (fabs(sum) >= fabs(v))
        comp += (sum - t) + v;
    else
        comp += (v - t) + sum;
    sum = t;
}

// ---- sorted-entry PARITY reduction -------------------------------------------------------
// Every fraction entry (cell c, slot e) becomes a 64-bit key (particle index << 32 | c << 1 |
// e). The entries are emitted in lexicographic cell order (a tiled scan over the count field:
// per-tile entry totals, a scan over tiles, then each tile writes its entries in order), so a
// STABLE radix sort on the particle bits alone — two 8-bit passes for up to 65k particles —
// leaves each particle's entries in finalize_hydro_forces' visiting order (cells
// lexicographic, entry 0 before 1, psm.cpp:288-308). Six threads per particle (f.x f.y f.z
// t.x t.y t.z) then run the Neumaier chains over the particle's segment. No walk over empty
// cells, any fraction field.
constexpr int kEntryThreads = 256;
constexpr int kEntryPerThread = 16;
constexpr int kEntryTile = kEntryThreads * kEntryPerThread;

__global__ void __launch_bounds__(kEntryThreads) entry_tile_sums_kernel(const uint8_t* __restrict__ count,
                                                                        long long cells, int* __restrict__ sums) {
    using Reduce = cub::BlockReduce<int, kEntryThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const long long c0 = (long long)blockIdx.x * kEntryTile + (long long)threadIdx.x * kEntryPerThread;
    int n = 0;
#pragma unroll
    for (int t = 0; t < kEntryPerThread; ++t)
        if (c0 + t < cells) n += count[c0 + t];
    const int total = Reduce(tmp).Sum(n);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kEntryThreads) entry_emit_kernel(
    const uint8_t* __restrict__ count, long long cells, const int* __restrict__ tile_off,
    const int* __restrict__ id0, const int* __restrict__ id1, SnapIndex sidx, int n_snaps,
    unsigned long long* __restrict__ keys, DeviceErrors* err) {
    using Scan = cub::BlockScan<int, kEntryThreads>;
    __shared__ typename Scan::TempStorage tmp;
    const long long c0 = (long long)blockIdx.x * kEntryTile + (long long)threadIdx.x * kEntryPerThread;
    int cnt[kEntryPerThread];
    int n = 0;
#pragma unroll
    for (int t = 0; t < kEntryPerThread; ++t) {
        cnt[t] = c0 + t < cells ? count[c0 + t] : 0;
        n += cnt[t];
    }
    int off = 0;
    Scan(tmp).ExclusiveSum(n, off);
    unsigned long long* out = keys + tile_off[blockIdx.x] + off;
    for (int t = 0; t < kEntryPerThread; ++t) {
        const long long c = c0 + t;
        for (int e = 0; e < cnt[t]; ++e) {
            int p = sidx(e == 0 ? id0[c] : id1[c]);
            if (p < 0) {
                atomicAdd(&err->unknown, 1ull);
                p = n_snaps;  // sorts last, outside every particle's segment
            }
            *out++ = ((unsigned long long)p << 32) | ((unsigned long long)c << 1) | (unsigned long long)e;
        }
    }
}

__global__ void __launch_bounds__(256) segment_kernel(const unsigned long long* __restrict__ keys, long long n,
                                                      int n_snaps, int* __restrict__ start, int* __restrict__ end) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned p = (unsigned)(keys[i] >> 32);
    if (p >= (unsigned)n_snaps) return;  // unknown id (SyncError is raised)
    if (i == 0 || (unsigned)(keys[i - 1] >> 32) != p) start[p] = (int)i;
    if (i == n - 1 || (unsigned)(keys[i + 1] >> 32) != p) end[p] = (int)(i + 1);
}

// One warp per particle. The warp loads 32 consecutive entries of the particle's segment at a
// time (coalesced keys, then the 32 momenta, all in flight together), each lane computes its
// entry's six terms (f = m, t = cross(c - x, m), psm.cpp:294-296) into shared memory, and lanes
// 0..5 — one per component — add the 32 terms in entry order with Neumaier steps (vec3.hpp:75-82),
// so each component's (sum, comp) is the reference's serial walk exactly. The next batch's
// momenta are gathered before the current batch is replayed, with their keys loaded one
// batch earlier still. (Clearing the scratch from here, by
// the loading lane, measured 10x slower than the separate clear_entries_kernel pass.)
constexpr int kChainWarps = 8;

__global__ void __launch_bounds__(32 * kChainWarps) chain_kernel(
    const unsigned long long* __restrict__ keys, const int* __restrict__ start, const int* __restrict__ end,
    const lbg_snapshot* __restrict__ s, int n_snaps, BinGeom g, const double* __restrict__ m0,
    const double* __restrict__ m1, double* __restrict__ rows, int* __restrict__ used, int fast) {
    __shared__ double terms[kChainWarps][32][7];  // padded row: lanes 0..5 read a column
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int p = blockIdx.x * kChainWarps + w;
    if (p >= n_snaps) return;  // warp-uniform
    const int i0 = start[p], i1 = end[p];
    const double x0 = s[p].x[0], x1 = s[p].x[1], x2 = s[p].x[2];
    double (*tw)[7] = terms[w];
    // software pipeline: the keys two batches ahead, the momenta one batch ahead, so neither
    // the key load nor the dependent momentum gather of a batch is waited on before its replay
    auto key_at = [&](int base) { return base + lane < i1 ? keys[base + lane] : 0ull; };
    auto gather = [&](int base, unsigned long long key, long long& c, double& a0, double& a1, double& a2) {
        if (base + lane < i1) {
            c = (long long)((key >> 1) & 0x7fffffffull);
            const double* mp = ((key & 1ull) ? m1 : m0) + 3 * c;
            a0 = mp[0];
            a1 = mp[1];
            a2 = mp[2];
        }
    };
    long long c = 0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    gather(i0, key_at(i0), c, a0, a1, a2);
    unsigned long long knext = key_at(i0 + 32);
    double sum = 0.0, comp = 0.0;
    for (int base = i0; base < i1; base += 32) {
        const int n = min(32, i1 - base);
        if (lane < n) {
            const int ci = (int)(c % g.dims[0]), cj = (int)((c / g.dims[0]) % g.dims[1]),
                      ck = (int)(c / ((long long)g.dims[0] * g.dims[1]));
            const double r0 = ((double)(g.lo[0] + ci) + 0.5) - x0;
            const double r1 = ((double)(g.lo[1] + cj) + 0.5) - x1;
            const double r2 = ((double)(g.lo[2] + ck) + 0.5) - x2;
            tw[lane][0] = a0;
            tw[lane][1] = a1;
            tw[lane][2] = a2;
            tw[lane][3] = r1 * a2 - r2 * a1;
            tw[lane][4] = r2 * a0 - r0 * a2;
            tw[lane][5] = r0 * a1 - r1 * a0;
        }
        __syncwarp();
        gather(base + 32, knext, c, a0, a1, a2);  // next batch's momenta in flight during the replay
        knext = key_at(base + 64);                  // and the keys of the batch after
        if (lane < 6) {
            for (int e = 0; e < n; ++e) {
                const double v = tw[e][lane];
                if (fast)
                    sum += v;
                else
                    nm_add(sum, comp, v);
            }
        }
        __syncwarp();
    }
    if (lane < 6) {
        const int slot = lane < 3 ? lane : 6 + (lane - 3);
        rows[12 * (size_t)p + slot] = sum;
        rows[12 * (size_t)p + slot + 3] = comp;
    }
    if (lane == 0) used[p] = i1 > i0;
}

// the reference clears the scratch of every visited entry (psm.cpp:305)
__global__ void __launch_bounds__(256) clear_entries_kernel(const unsigned long long* __restrict__ keys, long long n,
                                                            double* __restrict__ m0, double* __restrict__ m1) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long c = (long long)((keys[i] >> 1) & 0x7fffffffull);
    double* mp = ((keys[i] & 1ull) ? m1 : m0) + 3 * c;
    mp[0] = mp[1] = mp[2] = 0.0;
}

static BinGeom geom(lbg_block b) {
    BinGeom g;
    const int d[3] = {b->L.nx, b->L.ny, b->L.nz};
    for (int a = 0; a < 3; ++a) {
        g.dims[a] = d[a];
        g.lo[a] = b->lo[a];
        g.nb[a] = (d[a] + kBin - 1) / kBin;
    }
    return g;
}

__global__ void snap_table_kernel(const lbg_snapshot* __restrict__ s, int n, int id_min, int* __restrict__ tab) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) tab[s[p].id - id_min] = p;
}

static lbg_status upload_snapshots(lbg_block b, const lbg_snapshot* snaps, int n) {
    for (int t = 1; t < n; ++t)
        if (snaps[t].id <= snaps[t - 1].id)
            return set_error(LBG_INVALID, "snapshots must be sorted by ascending unique id");
    if (n > b->snaps_cap) {
        LBG_CUDA(cudaStreamSynchronize(b->side));
        LBG_CUDA(cudaStreamSynchronize(b->stream));
        if (b->snaps_h) cudaFreeHost(b->snaps_h);
        b->snaps_h = nullptr;
        const int cap = std::max(n, 2 * b->snaps_cap);
        b->snaps_cap = 0;
        LBG_CUDA(cudaMallocHost(&b->snaps_h, sizeof(lbg_snapshot) * cap));
        int dcap = 0;
        if (lbg_status s = grow_device(b->snaps_d, dcap, cap, cap, "cudaMalloc(snapshots)")) return s;
        b->snaps_cap = cap;
    }
    // staging buffer may still feed the previous copy
    LBG_CUDA(cudaEventSynchronize(b->ev_side));
    if (n > 0) std::memcpy(b->snaps_h, snaps, sizeof(lbg_snapshot) * n);
    // the previous step's kernels may still read snaps_d: order the copy after them
    LBG_CUDA(cudaEventRecord(b->ev_side, b->stream));
    LBG_CUDA(cudaStreamWaitEvent(b->side, b->ev_side, 0));
    if (n > 0)
        LBG_CUDA(cudaMemcpyAsync(b->snaps_d, b->snaps_h, sizeof(lbg_snapshot) * n,
                                 cudaMemcpyHostToDevice, b->side));
    LBG_CUDA(cudaEventRecord(b->ev_side, b->side));
    LBG_CUDA(cudaStreamWaitEvent(b->stream, b->ev_side, 0));
    b->n_snaps = n;
    // dense id -> index table when the ids are dense (SnapIndex), on the compute stream
    b->snap_range = 0;
    if (n > 0) {
        const long long range = (long long)snaps[n - 1].id - snaps[0].id + 1;
        if (range <= 4LL * n + 4096) {
            if (lbg_status s = grow_device(b->snap_tab, b->snap_tab_cap, range, 2 * b->snap_tab_cap,
                                           "cudaMalloc(snapshot index)"))
                return s;
            b->snap_id_min = snaps[0].id;
            b->snap_range = (int)range;
            LBG_CUDA(cudaMemsetAsync(b->snap_tab, 0xff, sizeof(int) * range, b->stream));
            snap_table_kernel<<<(n + 255) / 256, 256, 0, b->stream>>>(b->snaps_d, n, b->snap_id_min, b->snap_tab);
            LBG_LAUNCH_CHECK();
        }
    }
    return LBG_OK;
}

static lbg_status ensure_bins(lbg_block b, long long nbins) {
    if (nbins <= b->n_bins_cap && b->bin_count && b->bin_start) return LBG_OK;
    b->n_bins_cap = 0;
    long long c1 = 0, c2 = 0;
    if (lbg_status s = grow_device(b->bin_count, c1, 2 * nbins, 2 * nbins, "cudaMalloc(bins)")) return s;  // count + cursor
    if (lbg_status s = grow_device(b->bin_start, c2, nbins + 1, nbins + 1, "cudaMalloc(bins)")) return s;
    b->n_bins_cap = nbins;
    return LBG_OK;
}

lbg_status rebuild_covered(lbg_block b) {
    const long long cells = (long long)b->L.nx * b->L.ny * b->L.nz;
    LBG_CUDA(cudaMemsetAsync(b->cov_n, 0, 2 * sizeof(int), b->stream));
    covered_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, b->stream>>>(b->count, cells, b->cov_n);
    LBG_LAUNCH_CHECK();
    const long long rows = (long long)b->L.ny * b->L.nz;
    const long long nseg = rows * ((b->L.nx + 31) / 32);
    LBG_CUDA(cudaMemsetAsync(b->seg_n, 0, 2 * sizeof(int), b->stream));
    segments_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, b->stream>>>(b->count, b->L.nx, rows, b->seg_list,
                                                                           b->seg_n, b->seg_cap);
    LBG_LAUNCH_CHECK();
    b->cov_dirty = false;
    return LBG_OK;
}

}  // namespace lbg

using namespace lbg;

static lbg_status need_coupling(lbg_block b) {
    if (!b) return set_error(LBG_INVALID, "null block");
    if (!b->coupling) return set_error(LBG_INVALID, "block was created without coupling fields");
    return LBG_OK;
}

// per-particle accumulators of LBG_FORCE_FUSED, zeroed once per step (at the mapping)
static lbg_status prepare_fused(lbg_block b, int n) {
    if (b->force_mode != LBG_FORCE_FUSED) return LBG_OK;
    if (n > b->facc_cap || !b->facc || !b->fused_used) {
        const int cap = std::max(n, std::max(1, 2 * b->facc_cap));
        b->facc_cap = 0;
        long long c1 = 0, c2 = 0;
        if (lbg_status s = grow_device(b->facc, c1, 6LL * cap, 6LL * cap, "cudaMalloc(fused)")) return s;
        if (lbg_status s = grow_device(b->fused_used, c2, cap, cap, "cudaMalloc(fused)")) return s;
        b->facc_cap = cap;
    }
    LBG_CUDA(cudaMemsetAsync(b->facc, 0, sizeof(double) * 6 * b->facc_cap, b->stream));
    LBG_CUDA(cudaMemsetAsync(b->fused_used, 0, sizeof(int) * b->facc_cap, b->stream));
    return LBG_OK;
}

extern "C" {

lbg_status lbg_set_force_mode(lbg_block b, int mode) {
    if (lbg_status s = need_coupling(b)) return s;
    if (mode != LBG_FORCE_SCRATCH && mode != LBG_FORCE_FUSED) return set_error(LBG_INVALID, "bad force mode");
    LBG_CUDA(cudaSetDevice(b->device));
    b->force_mode = mode;
    // takes effect at once: the accumulators exist (zeroed, sized for the current list)
    // before any sweep can run in the new mode
    return prepare_fused(b, b->n_snaps);
}

lbg_status lbg_map(lbg_block b, const lbg_snapshot* snaps, int n, int subdivisions) {
    if (lbg_status s = need_coupling(b)) return s;
    if (subdivisions < 1) return set_error(LBG_CONFIG_ERROR, "subdivisions must be >= 1");
    LBG_CUDA(cudaSetDevice(b->device));
    Span span(b, LBG_CAT_MAPPING);
    if (lbg_status s = upload_snapshots(b, snaps, n)) return s;
    if (lbg_status s = prepare_fused(b, n)) return s;
    const BinGeom g = geom(b);
    const long long nbins = (long long)g.nb[0] * g.nb[1] * g.nb[2];
    if (lbg_status s = ensure_bins(b, nbins)) return s;
    int* cnt = b->bin_count;
    int* cursor = b->bin_count + nbins;
    const long long cells = (long long)b->L.nx * b->L.ny * b->L.nz;
    {
        const long long threads = std::max(2 * nbins, (cells + 15) / 16);
        map_zero_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, b->stream>>>(
            cnt, 2 * nbins, b->bin_start, b->cov_n, b->seg_n, b->count, b->btot, cells);
        LBG_LAUNCH_CHECK();
    }
    if (n > 0) {
        bin_count_kernel<<<(n + 127) / 128, 128, 0, b->stream>>>(b->snaps_d, n, g, cnt);
        LBG_LAUNCH_CHECK();
    }
    // persistent scan workspace (no per-call allocation)
    size_t tmp_bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt, b->bin_start + 1, (int)nbins, b->stream);
    if (lbg_status s = grow_device(b->scan_tmp, b->scan_tmp_bytes, (long long)tmp_bytes, (long long)tmp_bytes,
                                   "cudaMalloc(scan_tmp)"))
        return s;
    cub::DeviceScan::InclusiveSum(b->scan_tmp, tmp_bytes, cnt, b->bin_start + 1, (int)nbins, b->stream);
    LBG_LAUNCH_CHECK();
    // host upper bound of the registrations (bins a particle's reach box can touch), so the
    // item list is sized without reading the scan back: the whole mapping stays asynchronous
    long long bound = 1;
    for (int p = 0; p < n; ++p) {
        long long nb = 1;
        for (int d = 0; d < 3; ++d)
            nb *= std::min<long long>(g.nb[d], (long long)((2.0 * (snaps[p].r + 0.5) + 4.0) / kBin) + 2);
        bound += nb;
    }
    if (lbg_status s = grow_device(b->bin_items, b->bin_items_cap, bound, 2 * b->bin_items_cap,
                                   "cudaMalloc(bin items)"))
        return s;
    if (n > 0) {
        bin_fill_kernel<<<(n + 127) / 128, 128, 0, b->stream>>>(b->snaps_d, n, g, b->bin_start, cursor,
                                                                b->bin_items);
        LBG_LAUNCH_CHECK();
        bin_sort_kernel<<<(unsigned)((nbins + 127) / 128), 128, 0, b->stream>>>(b->bin_start, cnt, (int)nbins,
                                                                                b->bin_items);
        LBG_LAUNCH_CHECK();
    }
    MapArgs a{};
    a.s = b->snaps_d;
    a.g = g;
    a.start = b->bin_start;
    a.cnt = cnt;
    a.items = b->bin_items;
    a.count = b->count;
    a.id0 = b->id0;
    a.id1 = b->id1;
    a.b0 = b->b0;
    a.b1 = b->b1;
    a.btot = b->btot;
    a.v0 = b->v0;
    a.v1 = b->v1;
    a.err = b->err_d;
    a.cov_n = b->cov_n;
    // count and btot of every cell were zeroed by map_zero_kernel, so the mapping kernel skips
    // bins without candidates and writes only covered cells
    map_bin_kernel<<<(unsigned)nbins, 256, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
    const long long rows = (long long)b->L.ny * b->L.nz;
    const long long nseg = rows * ((b->L.nx + 31) / 32);
    segments_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, b->stream>>>(b->count, b->L.nx, rows, b->seg_list,
                                                                           b->seg_n, b->seg_cap);
    LBG_LAUNCH_CHECK();
    b->cov_dirty = false;
    b->v_snap = true;
    b->map_ids.resize(n);
    for (int p = 0; p < n; ++p) b->map_ids[p] = snaps[p].id;
    b->map_ids_valid = true;
    return LBG_OK;
}

// setu_kernel over the current fraction field with the current snapshots (psm.cpp:138-169)
static lbg_status run_setu(lbg_block b) {
    const BinGeom g = geom(b);
    dim3 grid((g.dims[0] + 127) / 128, g.dims[1], g.dims[2]);
    setu_kernel<<<grid, 128, 0, b->stream>>>(b->snaps_d, snap_index(b), g, b->count, b->id0, b->id1, b->v0, b->v1,
                                            b->err_d);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

// write the v_snap velocities into v0/v1 (before they are read or partly overwritten)
static lbg_status materialize_velocity(lbg_block b) {
    if (!b->v_snap) return LBG_OK;
    return run_setu(b);
}

lbg_status lbg_set_solid_velocities(lbg_block b, const lbg_snapshot* snaps, int n) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    Span span(b, LBG_CAT_SETU);
    if (lbg_status s = upload_snapshots(b, snaps, n)) return s;
    // every entry of a mapped field names a snapshot of the mapping list; if the new list
    // (id-sorted, like it) holds all of those ids, no entry can be unknown (psm.cpp:165-168)
    // and the PSM kernels evaluate u + omega x (c - x) from these snapshots inline. Otherwise
    // the field is filled here, counting unknown ids for lbg_sync's SyncError.
    bool superset = b->map_ids_valid;
    for (size_t p = 0, q = 0; superset && p < b->map_ids.size(); ++p) {
        while (q < (size_t)n && snaps[q].id < b->map_ids[p]) ++q;
        superset = q < (size_t)n && snaps[q].id == b->map_ids[p];
    }
    // fused force mode: the accumulators are indexed by this list's snapshot indices from
    // now on (the PSM sweep follows in the same step, sim.cpp:296-302): size and zero them
    if (lbg_status s = prepare_fused(b, n)) return s;
    if (superset) {  // nothing on the device can fail: the caller need not synchronise
        b->v_snap = true;
        return LBG_OK;
    }
    b->v_snap = false;
    if (lbg_status s = run_setu(b)) return s;
    // the exact walk ran: report its unknown-id count here, as set_solid_velocities throws
    // SyncError itself (psm.cpp:165-168)
    return lbg_sync(b, nullptr);
}

// LBG_FORCE_FUSED: the sweep already summed; copy the accumulators out
// per-particle output rows (device + pinned host), grown geometrically, kept across steps
static lbg_status reserve_rows(lbg_block b, int n) {
    const int need = std::max(n, 1);
    if (need <= b->red_cap) return LBG_OK;
    const int cap = std::max(need, 2 * b->red_cap);
    b->red_cap = 0;  // set again only when all four buffers exist
    long long c1 = 0, c2 = 0;
    if (lbg_status s = grow_device(b->red_rows, c1, 12LL * cap, 12LL * cap, "cudaMalloc(partials)")) return s;
    if (lbg_status s = grow_device(b->red_used, c2, cap, cap, "cudaMalloc(partials)")) return s;
    if (b->red_rows_h) cudaFreeHost(b->red_rows_h);
    if (b->red_used_h) cudaFreeHost(b->red_used_h);
    b->red_rows_h = nullptr;
    b->red_used_h = nullptr;
    LBG_CUDA(cudaMallocHost(&b->red_rows_h, sizeof(double) * 12 * cap));
    LBG_CUDA(cudaMallocHost(&b->red_used_h, sizeof(int) * cap));
    b->red_cap = cap;
    return LBG_OK;
}

static lbg_status reduce_fused(lbg_block b, lbg_hydro_partial* out, int capacity, int* n_out) {
    const int n = b->n_snaps;
    if (n > b->facc_cap || (n > 0 && !b->facc))
        return set_error(LBG_INVALID, "fused force accumulators smaller than the snapshot list");
    if (lbg_status s = reserve_rows(b, n)) return s;
    double* acc = b->red_rows_h;  // pinned: 6 per particle
    int* used = b->red_used_h;
    {
        Span span(b, LBG_CAT_REDF);
        if (n > 0) {
            LBG_CUDA(cudaMemcpyAsync(acc, b->facc, sizeof(double) * 6 * n, cudaMemcpyDeviceToHost, b->stream));
            LBG_CUDA(cudaMemcpyAsync(used, b->fused_used, sizeof(int) * n, cudaMemcpyDeviceToHost, b->stream));
        }
    }
    if (lbg_status s = lbg_sync(b, nullptr)) {
        if (s == LBG_SYNC_ERROR) return set_error(LBG_SYNC_ERROR, "hydrodynamic force for unknown particle id");
        return s;
    }
    int m = 0;
    for (int p = 0; p < n; ++p) {
        if (!used[p]) continue;
        if (m >= capacity) return set_error(LBG_INVALID, "hydro partial output capacity too small");
        lbg_hydro_partial& h = out[m++];
        h.id = b->snaps_h[p].id;
        for (int d = 0; d < 3; ++d) {
            h.f[d] = acc[6 * (size_t)p + d];
            h.t[d] = acc[6 * (size_t)p + 3 + d];
            h.f_comp[d] = 0.0;
            h.t_comp[d] = 0.0;
        }
    }
    if (n_out) *n_out = m;
    return LBG_OK;
}

lbg_status lbg_reduce_hydro(lbg_block b, int mode, lbg_hydro_partial* out, int capacity, int* n_out) {
    if (lbg_status s = need_coupling(b)) return s;
    if (n_out) *n_out = 0;
    if (b->force_mode == LBG_FORCE_FUSED) {
        if (mode != LBG_REDUCE_FAST)
            return set_error(LBG_INVALID, "PARITY reduction needs LBG_FORCE_SCRATCH (the fused sweep "
                                          "does not keep per-cell momenta)");
        LBG_CUDA(cudaSetDevice(b->device));
        return reduce_fused(b, out, capacity, n_out);
    }
    LBG_CUDA(cudaSetDevice(b->device));
    const int n = b->n_snaps;
    if (lbg_status s = reserve_rows(b, n)) return s;
    const BinGeom g = geom(b);
    const long long cells = (long long)g.dims[0] * g.dims[1] * g.dims[2];
    if (b->cov_dirty)
        if (lbg_status s = rebuild_covered(b)) return s;
    {
        Span span(b, LBG_CAT_REDF);
        if (!b->cn_h) LBG_CUDA(cudaMallocHost(&b->cn_h, 2 * sizeof(int)));  // pinned: no staged copy
        LBG_CUDA(cudaMemcpyAsync(b->cn_h, b->cov_n, 2 * sizeof(int), cudaMemcpyDeviceToHost, b->stream));
        LBG_CUDA(cudaStreamSynchronize(b->stream));
        const int cn[2] = {b->cn_h[0], b->cn_h[1]};
        const long long ne = (long long)cn[0] + 2LL * cn[1];
        if (!b->ekeys[0] || !b->ekeys[1] || !b->sort_tmp) {
            // sized once for the worst case (two entries per cell): steady-state steps never
            // allocate (cudaFree/cudaMalloc serialise all block-worker threads of a process)
            const long long cap = std::max(2 * cells, 1LL);
            long long c1 = 0, c2 = 0;
            if (lbg_status s = grow_device(b->ekeys[0], c1, cap, cap, "cudaMalloc(entry keys)")) return s;
            if (lbg_status s = grow_device(b->ekeys[1], c2, cap, cap, "cudaMalloc(entry keys)")) return s;
            b->ekeys_cap = cap;
            size_t tmp = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tmp, b->ekeys[0], b->ekeys[1], (int)cap, 0, 64, b->stream);
            if (lbg_status s = grow_device(b->sort_tmp, b->sort_tmp_bytes, (long long)tmp, (long long)tmp,
                                           "cudaMalloc(sort workspace)"))
                return s;
        }
        if (std::max(n, 1) > b->red_seg_cap || !b->red_seg) {
            const int cap = std::max(std::max(n, 1), 2 * b->red_seg_cap);
            int c1 = 0;
            b->red_seg_cap = 0;
            if (lbg_status s = grow_device(b->red_seg, c1, 2LL * cap, 2LL * cap, "cudaMalloc(segments)")) return s;
            b->red_seg_cap = cap;
        }
        if (ne > 0) {
            const long long tiles = (cells + kEntryTile - 1) / kEntryTile;
            if (tiles > b->tile_cap || !b->tile_buf) {
                long long c1 = 0;
                b->tile_cap = 0;
                if (lbg_status s = grow_device(b->tile_buf, c1, 2 * tiles, 2 * tiles, "cudaMalloc(entry tiles)"))
                    return s;
                b->tile_cap = tiles;
            }
            int* sums = b->tile_buf;
            int* offs = b->tile_buf + b->tile_cap;
            entry_tile_sums_kernel<<<(unsigned)tiles, kEntryThreads, 0, b->stream>>>(b->count, cells, sums);
            LBG_LAUNCH_CHECK();
            size_t tmp = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tmp, sums, offs, (int)tiles, b->stream);
            if (lbg_status s = grow_device(b->scan_tmp, b->scan_tmp_bytes, (long long)tmp, (long long)tmp,
                                           "cudaMalloc(scan_tmp)"))
                return s;
            cub::DeviceScan::ExclusiveSum(b->scan_tmp, tmp, sums, offs, (int)tiles, b->stream);
            entry_emit_kernel<<<(unsigned)tiles, kEntryThreads, 0, b->stream>>>(
                b->count, cells, offs, b->id0, b->id1, snap_index(b), n, b->ekeys[0], b->err_d);
            LBG_LAUNCH_CHECK();
            // stable LSD sort on the particle-index bits only (unknown ids carry index n)
            int bits = 1;
            while ((1ll << bits) < n + 1) ++bits;
            tmp = 0;
            cub::DeviceRadixSort::SortKeys(nullptr, tmp, b->ekeys[0], b->ekeys[1], (int)ne, 32, 32 + bits,
                                           b->stream);
            if (lbg_status s = grow_device(b->sort_tmp, b->sort_tmp_bytes, (long long)tmp, (long long)tmp,
                                           "cudaMalloc(sort_tmp)"))
                return s;
            cub::DeviceRadixSort::SortKeys(b->sort_tmp, tmp, b->ekeys[0], b->ekeys[1], (int)ne, 32, 32 + bits,
                                           b->stream);
            LBG_LAUNCH_CHECK();
        }
        if (n > 0) {
            int* start = b->red_seg;
            int* end = b->red_seg + b->red_seg_cap;
            LBG_CUDA(cudaMemsetAsync(start, 0, sizeof(int) * n, b->stream));
            LBG_CUDA(cudaMemsetAsync(end, 0, sizeof(int) * n, b->stream));
            if (ne > 0) {
                segment_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, b->stream>>>(b->ekeys[1], ne, n, start, end);
                LBG_LAUNCH_CHECK();
            }
            chain_kernel<<<(unsigned)((n + kChainWarps - 1) / kChainWarps), 32 * kChainWarps, 0, b->stream>>>(
                b->ekeys[1], start, end, b->snaps_d, n, g, b->m0, b->m1, b->red_rows, b->red_used,
                mode == LBG_REDUCE_FAST);
            LBG_LAUNCH_CHECK();
            if (ne > 0) {
                clear_entries_kernel<<<(unsigned)((ne + 255) / 256), 256, 0, b->stream>>>(b->ekeys[1], ne, b->m0,
                                                                                         b->m1);
                LBG_LAUNCH_CHECK();
            }
            LBG_CUDA(cudaMemcpyAsync(b->red_rows_h, b->red_rows, sizeof(double) * 12 * n,
                                     cudaMemcpyDeviceToHost, b->stream));
            LBG_CUDA(cudaMemcpyAsync(b->red_used_h, b->red_used, sizeof(int) * n, cudaMemcpyDeviceToHost,
                                     b->stream));
        }
    }
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    if (lbg_status s = lbg_sync(b, nullptr)) {
        if (s == LBG_SYNC_ERROR)
            return set_error(LBG_SYNC_ERROR, "hydrodynamic force for unknown particle id");
        return s;
    }
    int m = 0;
    for (int p = 0; p < n; ++p) {
        if (!b->red_used_h[p]) continue;
        if (m >= capacity) return set_error(LBG_INVALID, "hydro partial output capacity too small");
        lbg_hydro_partial& h = out[m++];
        h.id = b->snaps_h[p].id;
        const double* r = b->red_rows_h + 12 * (size_t)p;
        for (int d = 0; d < 3; ++d) {
            h.f[d] = r[d];
            h.f_comp[d] = r[3 + d];
            h.t[d] = r[6 + d];
            h.t_comp[d] = r[9 + d];
        }
    }
    if (n_out) *n_out = m;
    return LBG_OK;
}

static lbg_status copy_frac(lbg_block b, bool up, uint8_t* count, int* id0, int* id1, double* b0, double* b1,
                            double* btot) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    const size_t n = (size_t)b->L.nx * b->L.ny * b->L.nz;
    const auto kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    struct P {
        void* d;
        void* h;
        size_t bytes;
    } ps[] = {{b->count, count, n}, {b->id0, id0, 4 * n}, {b->id1, id1, 4 * n},
              {b->b0, b0, 8 * n},   {b->b1, b1, 8 * n},   {b->btot, btot, 8 * n}};
    for (auto& p : ps) {
        if (!p.h) continue;
        LBG_CUDA(cudaMemcpyAsync(up ? p.d : p.h, up ? p.h : p.d, p.bytes, kind, b->stream));
    }
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

lbg_status lbg_upload_fraction(lbg_block b, const uint8_t* count, const int* id0, const int* id1,
                               const double* b0, const double* b1, const double* btot) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    // the stored velocities belong to the old field: materialise them, then they are plain data
    if (lbg_status s = materialize_velocity(b)) return s;
    b->v_snap = false;
    b->map_ids_valid = false;
    b->cov_dirty = true;
    return copy_frac(b, true, (uint8_t*)count, (int*)id0, (int*)id1, (double*)b0, (double*)b1, (double*)btot);
}

lbg_status lbg_download_fraction(lbg_block b, uint8_t* count, int* id0, int* id1, double* b0, double* b1,
                                 double* btot) {
    return copy_frac(b, false, count, id0, id1, b0, b1, btot);
}

static lbg_status copy_vec_pair(lbg_block b, bool up, double* d0, double* d1, double* h0, double* h1) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    const size_t bytes = sizeof(double) * 3 * (size_t)b->L.nx * b->L.ny * b->L.nz;
    const auto kind = up ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    if (h0) LBG_CUDA(cudaMemcpyAsync(up ? d0 : h0, up ? h0 : d0, bytes, kind, b->stream));
    if (h1) LBG_CUDA(cudaMemcpyAsync(up ? d1 : h1, up ? h1 : d1, bytes, kind, b->stream));
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

lbg_status lbg_upload_solid_velocity(lbg_block b, const double* v0, const double* v1) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = materialize_velocity(b)) return s;  // a null side keeps its values
    b->v_snap = false;
    return copy_vec_pair(b, true, b ? b->v0 : nullptr, b ? b->v1 : nullptr, (double*)v0, (double*)v1);
}
lbg_status lbg_download_solid_velocity(lbg_block b, double* v0, double* v1) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = materialize_velocity(b)) return s;
    return copy_vec_pair(b, false, b ? b->v0 : nullptr, b ? b->v1 : nullptr, v0, v1);
}
lbg_status lbg_upload_scratch(lbg_block b, const double* m0, const double* m1) {
    return copy_vec_pair(b, true, b ? b->m0 : nullptr, b ? b->m1 : nullptr, (double*)m0, (double*)m1);
}
lbg_status lbg_download_scratch(lbg_block b, double* m0, double* m1) {
    return copy_vec_pair(b, false, b ? b->m0 : nullptr, b ? b->m1 : nullptr, m0, m1);
}

}  // extern "C"
