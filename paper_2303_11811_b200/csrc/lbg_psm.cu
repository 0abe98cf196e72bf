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

#include <algorithm>
#include <chrono>
#include <cstdio>
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

// Bin lists: each bin's registrations get one contiguous slot range. The ranges are handed
// out by a warp-aggregated cursor (one atomic per 32 bins) instead of a prefix scan: where a
// bin's list sits does not matter, only its content, which bin_sort_kernel then puts in
// ascending snapshot-index (= id) order, so the candidate sequence is deterministic.
__global__ void __launch_bounds__(256) bin_alloc_kernel(const int* __restrict__ cnt, int nbins,
                                                        int* __restrict__ start, int* __restrict__ cursor) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int n = b < nbins ? cnt[b] : 0;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    int base = 0;
    if (lane == 31 && incl > 0) base = atomicAdd(cursor, incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (b < nbins) start[b] = base + incl - n;
}

// one warp per bin: rank sort (each item's rank = number of smaller items; the items are
// distinct snapshot indices), in shared memory for up to kSortSmem items, serially by lane 0
// beyond that (only pathological overlap puts > 1024 particles in one 8^3 bin)
constexpr int kSortWarps = 8;
constexpr int kSortSmem = 1024;

// the mapping's per-candidate record, in the bin's sorted order (one load per candidate when
// the mapping kernel stages a bin instead of a list load and a dependent snapshot load)
struct MapRec {
    double x[3];
    double r, fr;
    int id, idx;
};
static_assert(sizeof(MapRec) == 48, "MapRec layout");

__device__ __forceinline__ void put_rec(MapRec* __restrict__ rec, const lbg_snapshot* __restrict__ s, int ix) {
    const lbg_snapshot& p = s[ix];
    MapRec r;
    r.x[0] = p.x[0];
    r.x[1] = p.x[1];
    r.x[2] = p.x[2];
    r.r = p.r;
    r.fr = p.f_r;
    r.id = p.id;
    r.idx = ix;
    *rec = r;
}

__global__ void __launch_bounds__(32 * kSortWarps) bin_sort_kernel(const int* __restrict__ start,
                                                                   const int* __restrict__ cnt, int nbins,
                                                                   int* __restrict__ items,
                                                                   const lbg_snapshot* __restrict__ snaps,
                                                                   MapRec* __restrict__ rec) {
    __shared__ int buf[kSortWarps][kSortSmem];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kSortWarps + w;
    if (b >= nbins) return;  // warp-uniform
    const int n = cnt[b];
    if (n == 0) return;
    int* a = items + start[b];
    MapRec* r = rec + start[b];
    if (n == 1) {
        if (lane == 0) put_rec(r, snaps, a[0]);
        return;
    }
    if (n > kSortSmem) {
        if (lane == 0)
            for (int i = 1; i < n; ++i) {
                const int v = a[i];
                int j = i - 1;
                while (j >= 0 && a[j] > v) {
                    a[j + 1] = a[j];
                    --j;
                }
                a[j + 1] = v;
            }
        __syncwarp();
        for (int t = lane; t < n; t += 32) put_rec(r + t, snaps, a[t]);
        return;
    }
    int* sb = buf[w];
    for (int t = lane; t < n; t += 32) sb[t] = a[t];
    __syncwarp();
    for (int t = lane; t < n; t += 32) {
        const int v = sb[t];
        int rk = 0;
        for (int u = 0; u < n; ++u) rk += sb[u] < v;
        a[rk] = v;
        put_rec(r + rk, snaps, v);
    }
}

struct MapArgs {
    const lbg_snapshot* __restrict__ s;
    BinGeom g;
    const int* __restrict__ start;
    const int* __restrict__ cnt;
    const int* __restrict__ items;
    const MapRec* __restrict__ rec;    // the bins' candidate records (sorted like items)
    uint8_t* __restrict__ count;
    int* __restrict__ id0;
    int* __restrict__ id1;
    int* __restrict__ pidx0;
    double* __restrict__ b0;
    double* __restrict__ b1;
    double* __restrict__ btot;
    DeviceErrors* err;
    long long items_cap;
    long long cells;
};

// K3 mapping (psm.cpp:28-32 overlap_fraction, psm.cpp:93-136 per-cell entry rule): one warp
// per 8 x 4 x 8 column of an 8^3 bin (lane = 8 x 4 cells of a z-level, looping over the bin's
// 8 z-levels), no CTA barrier. The warp stages the bin's candidates (32 at a time, list = id
// order) in its own shared-memory slots — read by all lanes as broadcasts — and per z-level
// keeps only the candidates that can reach a cell centre of its 8 x 4 slab (ballot), visited
// in ascending order. The overlap test is overlap_fraction with two exact shortcuts on the
// squared distance d2 = (dx*dx + dy*dy) + dz*dz (the radicand the reference takes the root of):
//   d2 > (r + f_r)^2 (1 + 1e-9)      => eps <= 0 (skip), the rounding of the root and of
//                                       -(dist - r) + f_r is ~1e-16 relative, far inside the
//                                       margin;
//   d2 < (r + f_r - 1)^2 (1 - 1e-9)  => eps >= 1, which the clamp makes exactly 1.0.
// Every other candidate takes the reference's sqrt path, so count/ids/fractions are bitwise
// those of build_fraction_field. count and btot of every cell were zeroed before the launch
// (what the reference stores for an uncovered cell), so only covered cells are written.
constexpr int kMapWarps = 8;

// distance from x to the interval [lo, hi] of cell-centre coordinates, as |c - x| of its
// nearest member c is computed (c - x rounded; for x > hi, x - hi = -(hi - x) exactly)
__device__ __forceinline__ double axis_gap(double lo, double hi, double x) {
    return x < lo ? lo - x : (x > hi ? x - hi : 0.0);
}

struct MapCand {
    double x0[32], x1[32], x2[32], r[32], fr[32], out2[32], in2[32], gxy[32];
    int id[32], idx[32];
};

// stage candidates [base, base + m) of the bin list; gxy = the squared x/y gap between the
// candidate and the warp's 8 x 4 column of cell centres (the z-independent part of the cull)
__device__ __forceinline__ void stage_cands(const MapArgs& a, const int* list, int base, int m, int lane,
                                            double wx0, double wx1, double wy0, double wy1, MapCand& sc) {
    if (lane < m) {
        const int ix = list[LBG_IDX((list - a.items) + base + lane, a.items_cap, a.err) - (list - a.items)];
        const lbg_snapshot& p = a.s[ix];
        sc.idx[lane] = ix;
        sc.x0[lane] = p.x[0];
        sc.x1[lane] = p.x[1];
        sc.x2[lane] = p.x[2];
        sc.r[lane] = p.r;
        sc.fr[lane] = p.f_r;
        const double ro = p.r + p.f_r, ri = ro - 1.0;
        sc.out2[lane] = (ro * ro) * (1.0 + 1e-9);
        sc.in2[lane] = ri > 0.0 ? (ri * ri) * (1.0 - 1e-9) : -1.0;
        const double g0 = axis_gap(wx0, wx1, p.x[0]), g1 = axis_gap(wy0, wy1, p.x[1]);
        sc.gxy[lane] = g0 * g0 + g1 * g1;
        sc.id[lane] = p.id;
    }
    __syncwarp();
}

template <int kMinBlocks>
__global__ void __launch_bounds__(32 * kMapWarps, kMinBlocks) map_warp_kernel(const MapArgs a) {
    __shared__ MapCand cand_all[kMapWarps];
    const BinGeom& g = a.g;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long unit = (long long)blockIdx.x * kMapWarps + w;  // (bin, y half)
    const long long nbins = (long long)g.nb[0] * g.nb[1] * g.nb[2];
    if (unit >= 2 * nbins) return;  // warp-uniform
    const int b = (int)(unit >> 1), yh = (int)(unit & 1);
    const int n = a.cnt[b];
    if (n == 0) return;
    MapCand& sc = cand_all[w];
    const int* list = a.items + a.start[b];
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const int i = bx * kBin + (lane & 7), j = by * kBin + yh * 4 + (lane >> 3);
    const double cc0 = (double)(g.lo[0] + i) + 0.5, cc1 = (double)(g.lo[1] + j) + 0.5;
    // cell-centre box of the warp's slab: x 8, y 4 (z per level)
    const double wx0 = (double)(g.lo[0] + bx * kBin) + 0.5, wx1 = wx0 + 7.0;
    const double wy0 = (double)(g.lo[1] + by * kBin + yh * 4) + 0.5, wy1 = wy0 + 3.0;
    const bool inxy = i < g.dims[0] && j < g.dims[1];
    if (n <= 32) stage_cands(a, list, 0, n, lane, wx0, wx1, wy0, wy1, sc);
    unsigned long long overfull = 0;
    for (int zz = 0; zz < kBin; ++zz) {
        const int k = bz * kBin + zz;
        if (k >= g.dims[2]) break;  // warp-uniform
        const double cc2 = (double)(g.lo[2] + k) + 0.5;
        const long long c = inxy ? LBG_IDX(((long long)k * g.dims[1] + j) * g.dims[0] + i, a.cells, a.err) : 0;
        int cnt = 0;
        double sum = 0.0;
        bool over = false;
        for (int base = 0; base < n; base += 32) {
            const int m = min(32, n - base);
            if (n > 32) {
                __syncwarp();  // every lane is done with the previous chunk
                stage_cands(a, list, base, m, lane, wx0, wx1, wy0, wy1, sc);
            }
            // warp-level cull: the squared gap between the candidate and the slab's box of cell
            // centres bounds every cell's radicand from below in floating point too (each
            // per-axis gap is the smallest |c - x| over the box, rounding is monotonic), so
            // the box rejects only candidates every cell rejects (rad > out2)
            bool rl = false;
            if (lane < m) {
                const double g2 = axis_gap(cc2, cc2, sc.x2[lane]);
                rl = !(sc.gxy[lane] + g2 * g2 > sc.out2[lane]);  // (g0 g0 + g1 g1) + g2 g2
            }
            const unsigned rel = __ballot_sync(0xffffffffu, rl);
            if (!inxy || over) continue;
            for (unsigned mask = rel; mask; mask &= mask - 1) {  // ascending = id order
                const int q = __ffs(mask) - 1;
                const double d0 = cc0 - sc.x0[q], d1 = cc1 - sc.x1[q], d2 = cc2 - sc.x2[q];
                const double rad = (d0 * d0 + d1 * d1) + d2 * d2;
                if (rad > sc.out2[q]) continue;
                double eps;
                if (rad < sc.in2[q]) {
                    eps = 1.0;
                } else {
                    eps = -(sqrt(rad) - sc.r[q]) + sc.fr[q];
                    eps = eps < 0.0 ? 0.0 : (1.0 < eps ? 1.0 : eps);  // std::clamp
                    if (eps <= 0.0) continue;
                }
                if (cnt >= 2) {
                    over = true;
                    break;
                }
                if (cnt == 0) {
                    a.id0[c] = sc.id[q];
                    a.pidx0[c] = sc.idx[q];
                    a.b0[c] = eps;
                } else {
                    a.id1[c] = sc.id[q];
                    a.b1[c] = eps;
                }
                ++cnt;
                sum += eps;
            }
        }
        if (inxy && cnt > 0) {  // uncovered cells keep the zeroed count and btot (+0.0)
            a.count[c] = (uint8_t)cnt;
            a.btot[c] = sum < 1.0 ? sum : 1.0;  // std::min(1.0, sum)
        }
        overfull += (unsigned long long)__popc(__ballot_sync(0xffffffffu, inxy && over));
    }
    if (overfull && lane == 0) atomicAdd(&a.err->overfull, overfull);
}

// K3 (default): candidate-outer, one warp per unit. A unit is an 8 x 4 x 8 cell
// column of an occupied 8^3 bin (lane = 8 x 4 cells of a level), and each lane keeps the state
// of its 8 cells (one per z-level: count, running sum, overfull flag) in registers while the
// loop runs the bin's candidates outside and the levels inside. A cell still visits its
// candidates in ascending (id) order with the same operations — rad = (d0*d0 + d1*d1) + d2*d2,
// whose z-independent d0*d0 + d1*d1 is now computed once per candidate instead of once per
// level — so the entries are bitwise those of map_warp_kernel. The per-level cull (the
// column's x/y gap plus the level's z gap against (r + f_r)^2 (1 + 1e-9)) runs once per
// candidate at staging time (lane = candidate) into a bit mask of the levels it can reach.
// Candidates are staged from the bins' sorted records (one load instead of list -> snapshot).
// LBG_MAP_COL=0 selects map_warp_kernel.
struct MapCandZ {
    double x0[32], x1[32], x2[32], r[32], fr[32], out2[32], in2[32];
    int id[32], idx[32];
    unsigned zm[32];
};

__device__ __forceinline__ void stage_recs(const MapRec* rec, int m, int lane, double wx0, double wx1, double wy0,
                                           double wy1, double z0c, int nz, MapCandZ& sc) {
    if (lane < m) {
        const MapRec p = rec[lane];
        sc.idx[lane] = p.idx;
        sc.x0[lane] = p.x[0];
        sc.x1[lane] = p.x[1];
        sc.x2[lane] = p.x[2];
        sc.r[lane] = p.r;
        sc.fr[lane] = p.fr;
        const double ro = p.r + p.fr, ri = ro - 1.0;
        const double out2 = (ro * ro) * (1.0 + 1e-9);
        sc.out2[lane] = out2;
        sc.in2[lane] = ri > 0.0 ? (ri * ri) * (1.0 - 1e-9) : -1.0;
        const double g0 = axis_gap(wx0, wx1, p.x[0]), g1 = axis_gap(wy0, wy1, p.x[1]);
        const double gxy = g0 * g0 + g1 * g1;
        unsigned zm = 0;
        for (int zz = 0; zz < nz; ++zz) {
            const double cc2 = z0c + (double)zz;  // = (double)(lo + k) + 0.5 exactly
            const double g2 = axis_gap(cc2, cc2, p.x[2]);
            if (!(gxy + g2 * g2 > out2)) zm |= 1u << zz;
        }
        sc.zm[lane] = zm;
        sc.id[lane] = p.id;
    }
    __syncwarp();
}

// one unit (bin b, y half yh; the bin's n candidate records from `start`); returns the number
// of the warp's cells found overfull (lane 0's value counts)
__device__ __forceinline__ unsigned map_unit(const MapArgs& a, int b, int yh, int start, int n, int lane,
                                             MapCandZ& sc) {
    const BinGeom& g = a.g;
    const int bx = b % g.nb[0], by = (b / g.nb[0]) % g.nb[1], bz = b / (g.nb[0] * g.nb[1]);
    const int i = bx * kBin + (lane & 7), j = by * kBin + yh * 4 + (lane >> 3);
    const double cc0 = (double)(g.lo[0] + i) + 0.5, cc1 = (double)(g.lo[1] + j) + 0.5;
    const double wx0 = (double)(g.lo[0] + bx * kBin) + 0.5, wx1 = wx0 + 7.0;
    const double wy0 = (double)(g.lo[1] + by * kBin + yh * 4) + 0.5, wy1 = wy0 + 3.0;
    const int kz0 = bz * kBin;
    const int nz = min(kBin, g.dims[2] - kz0);
    const double z0c = (double)(g.lo[2] + kz0) + 0.5;
    const bool inxy = i < g.dims[0] && j < g.dims[1];
    const long long plane = (long long)g.dims[0] * g.dims[1];
    const long long c0 = inxy ? ((long long)kz0 * g.dims[1] + j) * g.dims[0] + i : 0;
    unsigned cnts = 0;  // 2 bits per level
    unsigned over = 0;  // 1 bit per level
    double sum[kBin];
#pragma unroll
    for (int zz = 0; zz < kBin; ++zz) sum[zz] = 0.0;
    for (int base = 0; base < n; base += 32) {
        const int m = min(32, n - base);
        __syncwarp();  // every lane is done with the previous chunk / unit
        stage_recs(a.rec + LBG_IDX((long long)start + base, a.items_cap, a.err), m, lane, wx0, wx1, wy0, wy1,
                   z0c, nz, sc);
        const unsigned rel = __ballot_sync(0xffffffffu, lane < m && sc.zm[lane] != 0u);
        if (!inxy) continue;
        for (unsigned mask = rel; mask; mask &= mask - 1) {  // ascending = id order
            const int q = __ffs(mask) - 1;
            const unsigned zm = sc.zm[q];
            const double d0 = cc0 - sc.x0[q], d1 = cc1 - sc.x1[q];
            const double dxy = d0 * d0 + d1 * d1;
            const double x2 = sc.x2[q], out2 = sc.out2[q], in2 = sc.in2[q];
#pragma unroll
            for (int zz = 0; zz < kBin; ++zz) {
                if (!((zm >> zz) & 1u)) continue;  // warp-uniform
                const double d2 = (z0c + (double)zz) - x2;
                const double rad = dxy + d2 * d2;
                if (rad > out2) continue;
                double eps;
                if (rad < in2) {
                    eps = 1.0;
                } else {
                    eps = -(sqrt(rad) - sc.r[q]) + sc.fr[q];
                    eps = eps < 0.0 ? 0.0 : (1.0 < eps ? 1.0 : eps);  // std::clamp
                    if (eps <= 0.0) continue;
                }
                if ((over >> zz) & 1u) continue;
                const unsigned cnt = (cnts >> (2 * zz)) & 3u;
                if (cnt >= 2) {
                    over |= 1u << zz;
                    continue;
                }
                const long long c = LBG_IDX(c0 + zz * plane, a.cells, a.err);
                if (cnt == 0) {
                    a.id0[c] = sc.id[q];
                    a.pidx0[c] = sc.idx[q];
                    a.b0[c] = eps;
                } else {
                    a.id1[c] = sc.id[q];
                    a.b1[c] = eps;
                }
                cnts += 1u << (2 * zz);
                sum[zz] += eps;
            }
        }
    }
#pragma unroll
    for (int zz = 0; zz < kBin; ++zz) {
        const unsigned cnt = (cnts >> (2 * zz)) & 3u;
        if (inxy && zz < nz && cnt > 0) {  // uncovered cells keep the zeroed count and btot (+0.0)
            const long long c = c0 + zz * plane;
            a.count[c] = (uint8_t)cnt;
            a.btot[c] = sum[zz] < 1.0 ? sum[zz] : 1.0;  // std::min(1.0, sum)
        }
    }
    return __reduce_add_sync(0xffffffffu, (unsigned)__popc(over));
}

// one warp per unit of every bin (empty bins exit), kWarps warps per CTA. Measured slower
// (profiles/r02_ab_k12.txt): a persistent grid over a list of the occupied bins' units (static
// or counter-driven) and a grid over that list — the bin-ordered grid keeps neighbouring bins,
// which write the same 128-byte lines, on one SM at one time.
template <int kWarps>
__global__ void __launch_bounds__(32 * kWarps, 32 / kWarps) map_col_kernel(const MapArgs a) {
    __shared__ MapCandZ cand_all[kWarps];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long unit = (long long)blockIdx.x * kWarps + w;
    const long long nbins = (long long)a.g.nb[0] * a.g.nb[1] * a.g.nb[2];
    if (unit >= 2 * nbins) return;  // warp-uniform
    const int b = (int)(unit >> 1);
    const int n = a.cnt[b];
    if (n == 0) return;
    const unsigned over = map_unit(a, b, (int)(unit & 1), a.start[b], n, lane, cand_all[w]);
    if (over && lane == 0) atomicAdd(&a.err->overfull, (unsigned long long)over);
}

// the zero fills of one mapping in one launch (instead of separate memsets, each an API call
// that the block-worker threads sharing a GPU serialise on): the bin counters and cursors, the
// slot cursor, the segment counters, and count (u8) + btot (+0.0) of every cell — what
// build_fraction_field stores for an uncovered cell (psm.cpp:128-129). T threads: thread t
// clears count bytes [16t, 16t + 16) (one uint4) and the btot double pairs t, t + T, ...,
// t + 7T, so every store instruction of a warp covers 512 contiguous bytes (a thread's own
// 128 bytes of btot would spread each warp store over 32 lines: 43 us per 2M cells instead
// of a few). `pairs` = cells / 2 double pairs exist; an odd last cell is cleared by thread 0.
__global__ void __launch_bounds__(256) map_zero_kernel(int* __restrict__ bins2, long long nbins2,
                                                       int* __restrict__ slot_cursor, int* __restrict__ seg_n,
                                                       uint8_t* __restrict__ count, double* __restrict__ btot,
                                                       long long cells, long long T) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nbins2) bins2[t] = 0;
    if (t < 2) seg_n[t] = 0;
    if (t == 0) *slot_cursor = 0;
    if (t >= T) return;
    const long long c0 = 16 * t;
    if (c0 + 16 <= cells) {
        reinterpret_cast<uint4*>(count)[t] = make_uint4(0u, 0u, 0u, 0u);
    } else {
        for (long long c = c0; c < cells; ++c) count[c] = 0;
    }
    const long long pairs = cells / 2;
    double2* bt = reinterpret_cast<double2*>(btot);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const long long i = t + u * T;
        if (i < pairs) bt[i] = make_double2(0.0, 0.0);
    }
    if (t == 0 && (cells & 1)) btot[cells - 1] = 0.0;
}

// segment lists from the count field (one thread per 32-cell row segment; warp-aggregated
// appends): one-entry-only segments from the front, segments with a two-entry cell from the back
__global__ void __launch_bounds__(256) segments_kernel(const uint8_t* __restrict__ count, int nx, long long rows,
                                                       unsigned* __restrict__ seg_list, int* __restrict__ seg_n,
                                                       long long seg_cap) {
    const int per_row = (nx + 31) / 32;
    const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int mx = 0;
    long long c0 = 0;
    if (s < rows * per_row) {
        const long long row = s / per_row;
        const int i0 = (int)(s % per_row) * 32;
        c0 = row * nx + i0;
        for (int i = 0; i < 32 && i0 + i < nx; ++i) mx = max(mx, (int)count[c0 + i]);
    }
    warp_append(mx == 1, (unsigned)c0, seg_list, &seg_n[0]);
    const unsigned m2 = __ballot_sync(0xffffffffu, mx >= 2);
    if (m2) {
        const int lane = threadIdx.x & 31, leader = __ffs(m2) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&seg_n[1], __popc(m2));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (mx >= 2) seg_list[seg_cap - 1 - (base + __popc(m2 & ((1u << lane) - 1)))] = (unsigned)c0;
    }
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

// ---- box-walk reduction (PARITY / FAST) -------------------------------------------------
// finalize_hydro_forces visits the cells in lexicographic order and, per entry, adds m and
// cross(c - x, m) into the entry particle's Neumaier sums (psm.cpp:278-322). A particle's
// entries all lie in a small cell box (its reach, or the box of its entries), and the
// lexicographic order restricted to that box is the box's own (k, j, i) order — so one warp
// per particle walks its box 32 cells at a time in that order, picks the cells whose entry 0 /
// entry 1 names the particle (entry 0 before entry 1 within a cell), stages their six terms in
// shared memory in walk order, and lanes 0..5 (f.x f.y f.z t.x t.y t.z) replay them with the
// reference's Neumaier steps: each (sum, comp) is the serial walk's exactly. The entry's
// scratch is zeroed once its value is consumed (the reference clears every visited entry,
// psm.cpp:305). No sort, no scan, no host round trip; FAST sums the same sequence plainly.
//   box source: the snapshot's reach (r + max(1/2, f_r), the mapping's candidate test) when
//   the fraction field was mapped from these positions; otherwise entry_box_kernel takes the
//   min/max cell of every particle's entries from the field itself (order-independent).
constexpr int kWalkWarps = 1;   // warps per CTA (one: register-limited residency is per warp)
constexpr int kWalkGroups = 4;  // particles per warp: lane groups of 8
constexpr int kWalkKeys = 256;  // entry keys staged per particle before a replay flush

struct WalkArgs {
    const lbg_snapshot* __restrict__ s;
    int n;
    BinGeom g;
    const uint8_t* __restrict__ count;
    const int* __restrict__ id0;
    const int* __restrict__ id1;
    double* __restrict__ m0;
    double* __restrict__ m1;
    const int* __restrict__ box;  // 6 per particle (-lo xyz, hi xyz) or null: reach box
    double* __restrict__ rows;
    int* __restrict__ used;
    int fast;
    DeviceErrors* err;
    long long cells;
};

// vec3.hpp:75-82 without a branch: the larger-magnitude operand first, as the reference's if
__device__ __forceinline__ void nm_add_sel(double& sum, double& comp, double v) {
    const double t = sum + v;
    const bool a = fabs(sum) >= fabs(v);
    const double big = a ? sum : v, small = a ? v : sum;
    comp += (big - t) + small;
    sum = t;
}

// four cells of one lane per walk step (cell t = step * 32 + u * 8 + lane-in-group)
struct WalkQuad {
    long long c[4];
    int cnt[4], e0[4], e1[4];
};

// One warp walks four particles, one per 8-lane group (so the six Neumaier chains of each
// particle run in lanes 0..5 of its group and every replay instruction serves four particles).
// Pass 1 walks each particle's box 32 cells per step (4 per lane, the next step's cell fields
// in flight) and stages the keys (cell << 1 | entry) of the particle's entries in walk order —
// only count and ids are read; pass 2 (whenever a group's stage nears full, and at the end)
// gathers the momenta 32 per group at a time, writes the six terms of each entry, zeroes the
// entry's scratch (psm.cpp:305), and lanes 0..5 of each group replay them in order.
// register cap: 128 (the natural 125; default) or 120 (17 resident warps per SM, so a
// 10^4-particle block fits one wave: measured no faster, 275 vs 263 us on config 3)
// kRows (LBG_WALK_ROWS=1; rows of at most 16 cells: every box of the reach path for r + f_r
// below 6.5, checked on the host): each lane of a group takes a whole box row, loads its
// cells' fields at once, and a group prefix over the lanes (rows in order) places the row's
// keys. Fewer instructions than the cell walk but a full load latency per row step: measured
// slower on config 3 (432 vs 263 us), so the cell walk is the default.
// kGroups: particles per warp (4 groups of 8 lanes, default; or 1 group of 32 lanes, for
// blocks whose particles do not fill the GPU: a quarter of the walk steps per particle, so the
// latency-bound chain of dependent cell loads is 4x shorter where there are too few warps to
// hide it; the replay then serves one particle per instruction).
template <int kRegs, bool kRows, int kKeys, int kGroups = kWalkGroups>
__global__ void __maxnreg__(kRegs) walk_chain_kernel(const WalkArgs a) {
    constexpr int kL = 32 / kGroups;  // lanes per particle
    constexpr int kBatch = 4 * kL;    // entries per replay batch (4 per lane)
    __shared__ unsigned keys_all[kWalkWarps][kGroups][kKeys];
    __shared__ double terms_all[kWalkWarps][kGroups][kBatch][7];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / kL, gl = lane % kL;
    const long long pw = (long long)(blockIdx.x * kWalkWarps + w) * kGroups;
    if (pw >= a.n) return;  // warp-uniform
    const int p = (int)pw + grp;
    const bool valid = p < a.n;
    unsigned* kb = keys_all[w][grp];
    double (*tw)[7] = terms_all[w][grp];
    const BinGeom& g = a.g;
    int id = -2;
    double x0 = 0.0, x1 = 0.0, x2 = 0.0;
    int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
    if (valid) {
        const lbg_snapshot& sp = a.s[p];
        id = sp.id;
        x0 = sp.x[0];
        x1 = sp.x[1];
        x2 = sp.x[2];
        if (a.box) {
            for (int d = 0; d < 3; ++d) {
                lo[d] = -a.box[6 * p + d];
                hi[d] = a.box[6 * p + 3 + d];
            }
        } else {
            // every cell with eps > 0 has |c - x| < r + f_r (psm.cpp:28-32), c = lo + i + 1/2:
            // the cells within R = r + max(1/2, f_r) of x per axis, one cell of margin
            const double R = sp.r + (sp.f_r > 0.5 ? sp.f_r : 0.5);
            const double xs[3] = {x0, x1, x2};
            for (int d = 0; d < 3; ++d) {
                const double o = xs[d] - (double)g.lo[d] - 0.5;
                lo[d] = max((int)ceil(o - R) - 1, 0);
                hi[d] = min((int)floor(o + R) + 1, g.dims[d] - 1);
            }
        }
    }
    const bool nonempty = hi[0] >= lo[0] && hi[1] >= lo[1] && hi[2] >= lo[2];
    const int ex = nonempty ? hi[0] - lo[0] + 1 : 1, ey = nonempty ? hi[1] - lo[1] + 1 : 1;
    const long long total = nonempty ? (long long)ex * ey * (hi[2] - lo[2] + 1) : 0;
    const unsigned gmask = kL == 32 ? 0xffffffffu : ((1u << kL) - 1u) << (kL * grp);
    const unsigned lt = ((1u << lane) - 1u) & gmask;
    double sum = 0.0, comp = 0.0;
    bool any = false;
    int nk = 0;

    // keys: box-local (di, dj, dk) packed in 10 bits each when the box allows (no division to
    // recover the cell in pass 2), else the cell index
    const bool packed = ex <= 1024 && ey <= 1024 && hi[2] - lo[2] + 1 <= 1024;
    // each lane's next cells (t = step * kBatch + u * kL + lane-in-group) as running
    // coordinates: fetch() is called for consecutive steps and advances them by kBatch cells
    int ci[4], cj[4], ck[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const unsigned tu = (unsigned)(u * kL + gl), r = tu / (unsigned)ex;
        ci[u] = lo[0] + (int)(tu - r * (unsigned)ex);
        cj[u] = lo[1] + (int)(r % (unsigned)ey);
        ck[u] = lo[2] + (int)(r / (unsigned)ey);
    }
    auto fetch = [&](long long step, WalkQuad& q) {
        (void)step;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            q.cnt[u] = 0;
            q.c[u] = 0;
            q.e0[u] = q.e1[u] = -1;
            if (nonempty && ck[u] <= hi[2]) {
                const long long c =
                    LBG_IDX(((long long)ck[u] * g.dims[1] + cj[u]) * g.dims[0] + ci[u], a.cells, a.err);
                q.cnt[u] = a.count[c];
                q.e0[u] = a.id0[c];
                q.e1[u] = a.id1[c];
                q.c[u] = packed ? (((long long)(ck[u] - lo[2]) << 20) | ((cj[u] - lo[1]) << 10) | (ci[u] - lo[0])) : c;
                ci[u] += kBatch;
                while (ci[u] > hi[0]) {
                    ci[u] -= ex;
                    if (++cj[u] > hi[1]) {
                        cj[u] = lo[1];
                        ++ck[u];
                    }
                }
            }
        }
    };
    // pass 2 over the staged keys of every group (lockstep batches; groups with fewer idle)
    auto flush = [&]() {
        __syncwarp();
        const int nb = (nk + kBatch - 1) / kBatch;
        const int nbmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)nb);
        long long gc[4];
        double gm[4][3];
        auto gather = [&](int b) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = b * kBatch + u * kL + gl;
                gc[u] = -1;
                gm[u][0] = gm[u][1] = gm[u][2] = 0.0;
                if (e < nk) {
                    const unsigned key = kb[e];
                    long long c;
                    if (packed) {
                        const unsigned v = key >> 1;
                        c = ((long long)(lo[2] + (int)(v >> 20)) * g.dims[1] + (lo[1] + (int)((v >> 10) & 1023u))) *
                                g.dims[0] +
                            (lo[0] + (int)(v & 1023u));
                    } else {
                        c = (long long)(key >> 1);
                    }
                    c = LBG_IDX(c, a.cells, a.err);
                    const double* mp = ((key & 1u) ? a.m1 : a.m0) + 3 * c;
                    gm[u][0] = mp[0];
                    gm[u][1] = mp[1];
                    gm[u][2] = mp[2];
                    gc[u] = packed ? (long long)key : ((c << 1) | (key & 1u));
                }
            }
        };
        gather(0);
        for (int b = 0; b < nbmax; ++b) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (gc[u] < 0) continue;
                int xi, xj, xk;
                long long cell;
                if (packed) {
                    const unsigned v = (unsigned)(gc[u] >> 1);
                    xi = lo[0] + (int)(v & 1023u);
                    xj = lo[1] + (int)((v >> 10) & 1023u);
                    xk = lo[2] + (int)(v >> 20);
                    cell = ((long long)xk * g.dims[1] + xj) * g.dims[0] + xi;
                } else {
                    cell = gc[u] >> 1;
                    const unsigned cu = (unsigned)cell, row = cu / (unsigned)g.dims[0];
                    xi = (int)(cu - row * (unsigned)g.dims[0]);
                    xj = (int)(row % (unsigned)g.dims[1]);
                    xk = (int)(row / (unsigned)g.dims[1]);
                }
                const double r0 = ((double)(g.lo[0] + xi) + 0.5) - x0;
                const double r1 = ((double)(g.lo[1] + xj) + 0.5) - x1;
                const double r2 = ((double)(g.lo[2] + xk) + 0.5) - x2;
                const double* m = gm[u];
                double* t = tw[u * kL + gl];
                t[0] = m[0];
                t[1] = m[1];
                t[2] = m[2];
                t[3] = r1 * m[2] - r2 * m[1];
                t[4] = r2 * m[0] - r0 * m[2];
                t[5] = r0 * m[1] - r1 * m[0];
                double* z = ((gc[u] & 1) ? a.m1 : a.m0) + 3 * cell;  // the visited entry is cleared
                z[0] = 0.0;
                z[1] = 0.0;
                z[2] = 0.0;
            }
            __syncwarp();
            const int ne = min(kBatch, nk - b * kBatch);
            gather(b + 1);  // the next batch's momenta in flight during the replay
            if (gl < 6) {
#pragma unroll 4
                for (int e = 0; e < ne; ++e) {
                    const double v = tw[e][gl];
                    if (a.fast)
                        sum += v;
                    else
                        nm_add_sel(sum, comp, v);
                }
            }
            __syncwarp();
        }
        nk = 0;
    };
    auto step = [&](const WalkQuad& q) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool h0 = q.cnt[u] >= 1 && q.e0[u] == id, h1 = q.cnt[u] >= 2 && q.e1[u] == id;
            const unsigned b0 = __ballot_sync(0xffffffffu, h0), b1 = __ballot_sync(0xffffffffu, h1);
            const int s0 = nk + __popc(b0 & lt) + __popc(b1 & lt);
            if (h0) kb[LBG_IDX(s0, kKeys, a.err)] = (unsigned)(q.c[u] << 1);
            if (h1) kb[LBG_IDX(s0 + (h0 ? 1 : 0), kKeys, a.err)] = (unsigned)((q.c[u] << 1) | 1);
            nk += __popc(b0 & gmask) + __popc(b1 & gmask);
            any = any || ((b0 | b1) & gmask) != 0;
        }
    };
    const long long steps = (total + kBatch - 1) / kBatch;
    long long smax = steps;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    if constexpr (kRows) {
        const int ez = nonempty ? hi[2] - lo[2] + 1 : 0;
        const int rows = nonempty ? ey * ez : 0;
        const int rsteps = (rows + 7) / 8;
        const int rsmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)rsteps);
        for (int rs = 0; rs < rsmax; ++rs) {
            const int r = rs * 8 + gl;
            const bool rv = r < rows;
            int j = 0, k = 0;
            if (rv) {
                j = lo[1] + (int)((unsigned)r % (unsigned)ey);
                k = lo[2] + (int)((unsigned)r / (unsigned)ey);
            }
            const long long c0 = ((long long)k * g.dims[1] + j) * g.dims[0] + lo[0];
            int cnt[16], f0[16], f1[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                cnt[u] = 0;
                f0[u] = f1[u] = -1;
                if (rv && u < ex) {
                    const long long c = LBG_IDX(c0 + u, a.cells, a.err);
                    cnt[u] = a.count[c];
                    f0[u] = a.id0[c];
                    f1[u] = a.id1[c];
                }
            }
            unsigned hm = 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                if (cnt[u] >= 1 && f0[u] == id) hm |= 1u << (2 * u);
                if (cnt[u] >= 2 && f1[u] == id) hm |= 1u << (2 * u + 1);
            }
            const int mine = __popc(hm);
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o, 8);
                if (gl >= o) incl += v;
            }
            const int gtotal = __shfl_sync(0xffffffffu, incl, 7, 8);
            int slot = nk + incl - mine;
            const unsigned rowkey = ((unsigned)(k - lo[2]) << 20) | ((unsigned)(j - lo[1]) << 10);
            while (hm) {  // the row's entries in (cell, entry) order
                const int bit = __ffs(hm) - 1;
                hm &= hm - 1;
                kb[LBG_IDX(slot++, kKeys, a.err)] = ((rowkey | (unsigned)(bit >> 1)) << 1) | (unsigned)(bit & 1);
            }
            nk += gtotal;
            any = any || gtotal > 0;
            if (__any_sync(0xffffffffu, nk > kKeys - 256)) flush();  // a row step adds <= 8 x 32
        }
        flush();
    } else {
    // two register quads swap roles (copying an in-flight load would wait for it); one flush
        // call site (the flush is most of the code: a second inlined copy would spill the
        // instruction cache), taken after every pair of steps that may have filled a stage
        WalkQuad A, B;
        fetch(0, A);
        for (long long st = 0;; st += 2) {
            if (st < smax) {
                fetch(st + 1, B);
                step(A);
            }
            if (st + 1 < smax) {
                fetch(st + 2, A);
                step(B);
            }
            const bool done = st + 2 >= smax;
            if (done || __any_sync(0xffffffffu, nk > kKeys - 4 * kBatch)) flush();  // 2 steps add <= 4 kBatch
            if (done) break;
        }
    }
    if (valid && gl < 6) {
        const int slot = gl < 3 ? gl : 6 + (gl - 3);
        a.rows[12 * (size_t)p + slot] = sum;
        a.rows[12 * (size_t)p + slot + 3] = comp;
    }
    if (valid && gl == 0) a.used[p] = any ? 1 : 0;
}

// generic box source: per particle the min/max cell of its entries (atomic max on -lo / hi:
// order-independent), warp-aggregated per particle; entries with an id missing from the
// snapshot list are counted (finalize_hydro_forces' SyncError, psm.cpp:300-303)
__global__ void __launch_bounds__(256) entry_box_kernel(const uint8_t* __restrict__ count, long long cells, int nx,
                                                        int ny, const int* __restrict__ id0,
                                                        const int* __restrict__ id1, SnapIndex sidx,
                                                        int* __restrict__ box, DeviceErrors* err) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int cnt = c < cells ? count[c] : 0;
    const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((long long)nx * ny));
    const int lane = threadIdx.x & 31;
    for (int e = 0; e < 2; ++e) {
        int p = -1;
        if (cnt > e) {
            p = sidx(e == 0 ? id0[c] : id1[c]);
            if (p < 0) atomicAdd(&err->unknown, 1ull);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, p);
        if (p < 0) continue;
        const int v[6] = {-i, -j, -k, i, j, k};
        int r[6];
        for (int d = 0; d < 6; ++d) r[d] = __reduce_max_sync(peers, (unsigned)(v[d] + 0x40000000)) - 0x40000000;
        if (lane == __ffs(peers) - 1)
            for (int d = 0; d < 6; ++d) atomicMax(&box[6 * p + d], r[d]);
    }
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
        b->snaps_cap = cap;
    }
    if (n > b->snaps_dcap || !b->snaps_d) {
        LBG_CUDA(cudaStreamSynchronize(b->stream));
        if (lbg_status s = grow_device(b->snaps_d, b->snaps_dcap, std::max(n, 1), std::max(b->snaps_cap, 1),
                                       "cudaMalloc(snapshots)"))
            return s;
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

// the covered-segment counts to the host (pinned, asynchronous) for the sweep's kernel choice
lbg_status post_segment_counts(lbg_block b) {
    if (!b->segn_h) LBG_CUDA(cudaMallocHost(&b->segn_h, 2 * sizeof(int)));
    if (!b->ev_segn) LBG_CUDA(cudaEventCreateWithFlags(&b->ev_segn, cudaEventDisableTiming));
    LBG_CUDA(cudaMemcpyAsync(b->segn_h, b->seg_n, 2 * sizeof(int), cudaMemcpyDeviceToHost, b->stream));
    LBG_CUDA(cudaEventRecord(b->ev_segn, b->stream));
    b->segn_pending = true;
    return LBG_OK;
}

lbg_status rebuild_covered(lbg_block b) {
    const long long rows = (long long)b->L.ny * b->L.nz;
    const long long nseg = rows * ((b->L.nx + 31) / 32);
    LBG_CUDA(cudaMemsetAsync(b->seg_n, 0, 2 * sizeof(int), b->stream));
    segments_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, b->stream>>>(b->count, b->L.nx, rows, b->seg_list,
                                                                           b->seg_n, b->seg_cap);
    LBG_LAUNCH_CHECK();
    b->cov_dirty = false;
    return post_segment_counts(b);
}

// the block's mapping state <-> the shadow (pointer swaps only)
void swap_map_state(lbg_block b) {
    MapState& m = *b->shadow;
    std::swap(b->count, m.count);
    std::swap(b->id0, m.id0);
    std::swap(b->id1, m.id1);
    std::swap(b->pidx0, m.pidx0);
    std::swap(b->b0, m.b0);
    std::swap(b->b1, m.b1);
    std::swap(b->btot, m.btot);
    std::swap(b->seg_list, m.seg_list);
    std::swap(b->seg_n, m.seg_n);
    std::swap(b->snaps_d, m.snaps_d);
    std::swap(b->snaps_dcap, m.snaps_dcap);
    std::swap(b->n_snaps, m.n_snaps);
    std::swap(b->snap_tab, m.snap_tab);
    std::swap(b->snap_tab_cap, m.snap_tab_cap);
    std::swap(b->snap_id_min, m.snap_id_min);
    std::swap(b->snap_range, m.snap_range);
    std::swap(b->map_ids, m.map_ids);
    std::swap(b->map_snaps, m.map_snaps);
    std::swap(b->map_ids_valid, m.map_ids_valid);
    std::swap(b->v_snap, m.v_snap);
    std::swap(b->p_direct, m.p_direct);
    std::swap(b->cov_dirty, m.cov_dirty);
}

lbg_status ensure_shadow(lbg_block b) {
    if (b->shadow) return LBG_OK;
    auto* m = new MapState;
    b->shadow = m;
    const size_t n = (size_t)b->L.nx * b->L.ny * b->L.nz + 64;
    struct A {
        void** p;
        size_t bytes;
    } allocs[] = {{(void**)&m->count, n},     {(void**)&m->id0, n * 4}, {(void**)&m->id1, n * 4},
                  {(void**)&m->pidx0, n * 4}, {(void**)&m->b0, n * 8},  {(void**)&m->b1, n * 8},
                  {(void**)&m->btot, n * 8},  {(void**)&m->seg_list, sizeof(unsigned) * (size_t)b->seg_cap},
                  {(void**)&m->seg_n, 2 * sizeof(int)}};
    for (auto& a : allocs) {
        LBG_CUDA(cudaMalloc(a.p, a.bytes));
        LBG_CUDA(cudaMemset(*a.p, 0, a.bytes));
        b->device_bytes += (long long)a.bytes;
    }
    LBG_CUDA(cudaMemset(m->id0, 0xff, n * 4));  // FractionField::resize (field.cpp:37-46)
    LBG_CUDA(cudaMemset(m->id1, 0xff, n * 4));
    return LBG_OK;
}

void free_shadow(lbg_block b) {
    MapState* m = b->shadow;
    if (!m) return;
    void* dev[] = {m->count, m->id0, m->id1, m->pidx0, m->b0, m->b1, m->btot, m->seg_list, m->seg_n,
                   m->snaps_d, m->snap_tab};
    for (void* p : dev)
        if (p) cudaFree(p);
    delete m;
    b->shadow = nullptr;
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
    b->prepared = false;
    Span span(b, LBG_CAT_MAPPING);
    if (lbg_status s = upload_snapshots(b, snaps, n)) return s;
    if (lbg_status s = prepare_fused(b, n)) return s;
    const BinGeom g = geom(b);
    const long long nbins = (long long)g.nb[0] * g.nb[1] * g.nb[2];
    if (lbg_status s = ensure_bins(b, nbins)) return s;
    int* cnt = b->bin_count;
    int* cursor = b->bin_count + nbins;
    int* slot_cursor = b->bin_start + nbins;
    const long long cells = (long long)b->L.nx * b->L.ny * b->L.nz;
    {
        const long long T = (cells + 15) / 16;  // 16 cells per thread (8 btot pairs)
        const long long threads = std::max(2 * nbins, T);
        map_zero_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, b->stream>>>(
            cnt, 2 * nbins, slot_cursor, b->seg_n, b->count, b->btot, cells, T);
        LBG_LAUNCH_CHECK();
    }
    if (n > 0) {  // an empty list leaves the zeroed field and empty segment lists
        // host upper bound of the registrations (bins a particle's reach box can touch), so
        // the item list is sized without a read-back: the whole mapping stays asynchronous
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
        if (lbg_status s = grow_device(b->bin_rec, b->bin_rec_cap, b->bin_items_cap, b->bin_items_cap,
                                       "cudaMalloc(bin records)"))
            return s;
        bin_count_kernel<<<(n + 127) / 128, 128, 0, b->stream>>>(b->snaps_d, n, g, cnt);
        LBG_LAUNCH_CHECK();
        bin_alloc_kernel<<<(unsigned)((nbins + 255) / 256), 256, 0, b->stream>>>(cnt, (int)nbins, b->bin_start,
                                                                                  slot_cursor);
        LBG_LAUNCH_CHECK();
        bin_fill_kernel<<<(n + 127) / 128, 128, 0, b->stream>>>(b->snaps_d, n, g, b->bin_start, cursor,
                                                                b->bin_items);
        LBG_LAUNCH_CHECK();
        bin_sort_kernel<<<(unsigned)((nbins + kSortWarps - 1) / kSortWarps), 32 * kSortWarps, 0, b->stream>>>(
            b->bin_start, cnt, (int)nbins, b->bin_items, b->snaps_d, b->bin_rec);
        LBG_LAUNCH_CHECK();
        MapArgs a{};
        a.s = b->snaps_d;
        a.g = g;
        a.start = b->bin_start;
        a.cnt = cnt;
        a.items = b->bin_items;
        a.rec = b->bin_rec;
        a.count = b->count;
        a.id0 = b->id0;
        a.id1 = b->id1;
        a.pidx0 = b->pidx0;
        a.b0 = b->b0;
        a.b1 = b->b1;
        a.btot = b->btot;
        a.err = b->err_d;
        a.items_cap = b->bin_items_cap;
        a.cells = cells;
        // count and btot of every cell were zeroed by map_zero_kernel, so the mapping kernel
        // skips bins without candidates and writes only covered cells
        const long long units = 2 * nbins;
        static const int minb = [] {  // LBG_MAP_MINB: 5 caps the registers at 48, 3 at 80 (A/B)
            const char* e = std::getenv("LBG_MAP_MINB");
            return e ? std::atoi(e) : 4;
        }();
        const unsigned mgrid = (unsigned)((units + kMapWarps - 1) / kMapWarps);
        static const int col = [] {  // LBG_MAP_COL=0: the level-outer kernel (A/B)
            const char* e = std::getenv("LBG_MAP_COL");
            return e ? std::atoi(e) : 1;
        }();
        static const int cw = [] {  // LBG_MAP_CTA_WARPS: 4 or 8 warps per CTA (A/B)
            const char* e = std::getenv("LBG_MAP_CTA_WARPS");
            return e && std::atoi(e) == 4 ? 4 : 8;
        }();
        if (col) {
            const unsigned grid = (unsigned)((units + cw - 1) / cw);
            cw == 4 ? map_col_kernel<4><<<grid, 128, 0, b->stream>>>(a) : map_col_kernel<8><<<grid, 256, 0, b->stream>>>(a);
        } else if (minb == 5) {
            map_warp_kernel<5><<<mgrid, 32 * kMapWarps, 0, b->stream>>>(a);
        } else {
            map_warp_kernel<4><<<mgrid, 32 * kMapWarps, 0, b->stream>>>(a);
        }
        LBG_LAUNCH_CHECK();
        const long long rows = (long long)b->L.ny * b->L.nz;
        const long long nseg = rows * ((b->L.nx + 31) / 32);
        segments_kernel<<<(unsigned)((nseg + 255) / 256), 256, 0, b->stream>>>(b->count, b->L.nx, rows,
                                                                               b->seg_list, b->seg_n, b->seg_cap);
        LBG_LAUNCH_CHECK();
    }
    if (!b->preparing)  // a prepared mapping posts its counts when committed
        if (lbg_status s = post_segment_counts(b)) return s;
    b->cov_dirty = false;
    b->v_snap = true;
    b->p_direct = true;
    b->map_ids.resize(n);
    for (int p = 0; p < n; ++p) b->map_ids[p] = snaps[p].id;
    b->map_ids_valid = true;
    b->map_snaps.assign(snaps, snaps + n);
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

lbg_status lbg_map_prepare(lbg_block b, const lbg_snapshot* snaps, int n, int subdivisions) {
    if (lbg_status s = need_coupling(b)) return s;
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = ensure_shadow(b)) return s;
    b->prepared = false;
    swap_map_state(b);  // map into the shadow; the current state stays in use meanwhile
    b->preparing = true;
    const lbg_status st = lbg_map(b, snaps, n, subdivisions);
    b->preparing = false;
    swap_map_state(b);
    if (st != LBG_OK) return st;
    b->prepared = true;
    return LBG_OK;
}

lbg_status lbg_map_commit(lbg_block b) {
    if (lbg_status s = need_coupling(b)) return s;
    if (!b->prepared) return set_error(LBG_INVALID, "lbg_map_commit without lbg_map_prepare");
    // later work on the stream uses the new state; in-flight work holds the old pointers, and
    // the old state is only written again by the next prepare (stream order)
    swap_map_state(b);
    b->prepared = false;
    // the committed field's counts (the shadow's were never posted)
    LBG_CUDA(cudaSetDevice(b->device));
    return post_segment_counts(b);
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
    bool same = b->map_ids_valid && (size_t)n == b->map_ids.size();
    for (int p = 0; same && p < n; ++p) same = snaps[p].id == b->map_ids[p];
    b->p_direct = same;
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
    // LBG_REDUCE_PROFILE=1: host-side phase times of this call on stderr (A/B diagnostics)
    static const bool prof = [] {
        const char* e = std::getenv("LBG_REDUCE_PROFILE");
        return e && e[0] == '1';
    }();
    using clk = std::chrono::steady_clock;
    const auto t_0 = clk::now();
    auto t_reach = t_0, t_launch = t_0, t_sync = t_0;
    const int n = b->n_snaps;
    if (lbg_status s = reserve_rows(b, n)) return s;
    const BinGeom g = geom(b);
    const long long cells = (long long)g.dims[0] * g.dims[1] * g.dims[2];
    // reach boxes hold every entry when the field was mapped (lbg_map) from snapshots whose
    // ids, positions and radii the current list keeps; otherwise boxes from the field itself
    bool reach_ok = b->map_ids_valid && b->map_snaps.size() == b->map_ids.size();
    for (size_t p = 0, q = 0; reach_ok && p < b->map_snaps.size(); ++p) {
        const lbg_snapshot& ms = b->map_snaps[p];
        while (q < (size_t)n && b->snaps_h[q].id < ms.id) ++q;
        reach_ok = q < (size_t)n && b->snaps_h[q].id == ms.id;
        if (!reach_ok) break;
        const lbg_snapshot& cs = b->snaps_h[q];
        reach_ok = std::memcmp(ms.x, cs.x, sizeof(ms.x)) == 0 && std::memcmp(&ms.r, &cs.r, sizeof(double)) == 0 &&
                   std::memcmp(&ms.f_r, &cs.f_r, sizeof(double)) == 0;
    }
    t_reach = clk::now();
    {
        Span span(b, LBG_CAT_REDF);
        if (!b->ev_red) LBG_CUDA(cudaEventCreateWithFlags(&b->ev_red, cudaEventDisableTiming));
        WalkArgs a{};
        a.s = b->snaps_d;
        a.n = n;
        a.g = g;
        a.count = b->count;
        a.id0 = b->id0;
        a.id1 = b->id1;
        a.m0 = b->m0;
        a.m1 = b->m1;
        a.rows = b->red_rows;
        a.used = b->red_used;
        a.fast = mode == LBG_REDUCE_FAST;
        a.err = b->err_d;
        a.cells = cells;
        if (!reach_ok) {
            if (std::max(n, 1) > b->red_box_cap || !b->red_box) {
                const int cap = std::max(std::max(n, 1), 2 * b->red_box_cap);
                b->red_box_cap = 0;
                long long c1 = 0;
                if (lbg_status s = grow_device(b->red_box, c1, 6LL * cap, 6LL * cap, "cudaMalloc(particle boxes)"))
                    return s;
                b->red_box_cap = cap;
            }
            // empty boxes: -lo and hi start far below any cell index
            LBG_CUDA(cudaMemsetAsync(b->red_box, 0x80, sizeof(int) * 6 * std::max(n, 1), b->stream));
            if (cells > 0) {
                entry_box_kernel<<<(unsigned)((cells + 255) / 256), 256, 0, b->stream>>>(
                    b->count, cells, g.dims[0], g.dims[1], b->id0, b->id1, snap_index(b), b->red_box, b->err_d);
                LBG_LAUNCH_CHECK();
            }
            a.box = b->red_box;
        }
        if (n > 0) {
            const int per_cta = kWalkWarps * kWalkGroups;
            static const int regs = [] {  // LBG_WALK_REGS: 128 (natural) or 120 (A/B)
                const char* e = std::getenv("LBG_WALK_REGS");
                return e ? std::atoi(e) : 128;
            }();
            static const int rows_ok = [] {  // LBG_WALK_ROWS=1: the row walk where it applies (A/B;
                const char* e = std::getenv("LBG_WALK_ROWS");  // measured slower: 432 vs 263 us)
                return e && e[0] == '1';
            }();
            // the row walk needs every reach-box row within 16 cells: 2 R + 3 <= 16 with
            // R = r + max(1/2, f_r) (the box is x +- R widened by one cell each side)
            bool rows = rows_ok && reach_ok;
            for (int q = 0; rows && q < n; ++q) {
                const lbg_snapshot& sp = b->snaps_h[q];
                const double R = sp.r + (sp.f_r > 0.5 ? sp.f_r : 0.5);
                rows = 2.0 * R + 3.0 <= 16.0;
            }
            const unsigned grid = (unsigned)((n + per_cta - 1) / per_cta);
            // one particle per warp (32 lanes) for lists shorter than LBG_WALK_ONE_BELOW
            // (default 0: off): a 4x shorter chain of dependent cell loads per particle
            static const int one_below = [] {
                const char* e = std::getenv("LBG_WALK_ONE_BELOW");
                return e ? std::atoi(e) : 0;
            }();
            if (!rows && n < one_below)
                walk_chain_kernel<128, false, 1024, 1><<<(unsigned)((n + kWalkWarps - 1) / kWalkWarps), 32 * kWalkWarps, 0,
                                                          b->stream>>>(a);
            else if (rows)
                walk_chain_kernel<128, true, 512><<<grid, 32 * kWalkWarps, 0, b->stream>>>(a);
            else if (regs >= 128)
                walk_chain_kernel<128, false, kWalkKeys><<<grid, 32 * kWalkWarps, 0, b->stream>>>(a);
            else
                walk_chain_kernel<120, false, kWalkKeys><<<grid, 32 * kWalkWarps, 0, b->stream>>>(a);
            LBG_LAUNCH_CHECK();
            // partials D2H on the side stream (pinned), ordered after the walk by an event
            LBG_CUDA(cudaEventRecord(b->ev_red, b->stream));
            LBG_CUDA(cudaStreamWaitEvent(b->side, b->ev_red, 0));
            LBG_CUDA(cudaMemcpyAsync(b->red_rows_h, b->red_rows, sizeof(double) * 12 * n, cudaMemcpyDeviceToHost,
                                     b->side));
            LBG_CUDA(cudaMemcpyAsync(b->red_used_h, b->red_used, sizeof(int) * n, cudaMemcpyDeviceToHost, b->side));
        }
    }
    t_launch = clk::now();
    // lbg_sync waits for the side stream's copies and reads the error counters
    if (lbg_status s = lbg_sync(b, nullptr)) {
        if (s == LBG_SYNC_ERROR)
            return set_error(LBG_SYNC_ERROR, "hydrodynamic force for unknown particle id");
        return s;
    }
    t_sync = clk::now();
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
    if (prof) {
        auto us = [](clk::time_point a, clk::time_point c) {
            return std::chrono::duration<double, std::micro>(c - a).count();
        };
        std::fprintf(stderr, "lbg_reduce_hydro n=%d reach_check %.1f us, launch %.1f us, sync %.1f us, unpack %.1f us\n",
                     n, us(t_0, t_reach), us(t_reach, t_launch), us(t_launch, t_sync), us(t_sync, clk::now()));
    }
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
    b->p_direct = false;
    b->map_ids_valid = false;
    b->map_snaps.clear();
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
