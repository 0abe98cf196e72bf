// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — fused pull-stream + SRT (+PSM) collide sweep over a CellBox.
//   reference: collide_stream_impl (lbm.cpp:21-49), psm_collide_stream_impl (psm.cpp:218-262)
//
// Roofline: HBM-bound. Algorithmic bytes per lattice update (LUP): 19 f64 pulled + 19 f64
// stored = 304 B for the plain sweep; the coupled sweep adds the 1-byte count per cell and,
// per covered cell, 8 B btot + per entry (8 B b + 4 B id read, 24 B m written; the solid
// velocity u + omega x (c - x) is evaluated from the L2-resident snapshot list, v_snap).
//
// Kernels:
//   K1 sweep_box   — one CellBox, 3-D grid; thread x maps to global i with the chunk origin
//                    aligned to 32 cells, so a warp's loads/stores of a q-plane are two 128-B
//                    lines (the pulled x-neighbour costs one extra sector per warp, from L2).
//   K1 sweep_pair  — the same sweep with 128-bit accesses (two cells per lane), selected by
//                    LBG_SWEEP_PAIR=1; measured 2 % slower than sweep_box at 512^3.
//   K1 sweep_flat  — up to 8 boxes in one launch (the boundary_shell boxes, field.cpp:55-72).
//   K2 psm_seg     — the aligned 32-cell row segments that hold covered cells (count > 0),
//                    from the segment lists the mapping pass writes; K1 skips exactly those
//                    segments, so each DRAM sector is swept by one kernel. Segments with only
//                    one-entry cells run the pair-scheduled one-entry operator on every lane
//                    (fluid lanes with B = 0 when unforced) — by default in psm_seg_pipe, the
//                    register-pipelined loop that has the next segment's loads in flight
//                    (LBG_K2_MODE: 0 plain loop, 1 pipelined, 2 TMA-fed psm_seg_tma);
//                    segments with a two-entry cell the pair-scheduled two-entry operator
//                    (~124 registers); the fluid majority keeps the 70-register SRT kernel
//                    (the paper's fused A100 kernel ran at 196 registers, 12.5 % occupancy,
//                    PAPER.md:676).
//   sweep_flat_coupled — thin boxes of a coupled block (shell), one-entry and two-entry
//                    lanes in two launches.
// Periodic wrap: for axes in b->wrap the pull reads the wrapped interior cell directly
// (what fill_periodic_ghosts would have copied into the ghost slot), so a fully periodic
// single-GPU step is one launch with no ghost fill.
// Unstable cells (lbm.hpp:106) are counted with a warp ballot into the block's error
// counter; lbg_sync() raises NumericError like the reference does after the sweep.
#include "lbg_cell.cuh"
#include "lbg_internal.cuh"
#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace lbg {

struct SweepArgs {
    const double* __restrict__ src;
    double* __restrict__ dst;
    Layout L;
    double inv_tau;
    Force F;
    DeviceErrors* err;
    int wrap[3];
    // coupling (interior lexicographic)
    const uint8_t* __restrict__ count;
    const double* __restrict__ b0;
    const double* __restrict__ b1;
    const double* __restrict__ btot;
    const double* __restrict__ v0;
    const double* __restrict__ v1;
    double* __restrict__ m0;
    double* __restrict__ m1;
    const unsigned* __restrict__ seg_list;  // covered 32-cell row segments: max count 1 front, 2 back
    const int* __restrict__ seg_n;
    long long seg_cap;
    const int* __restrict__ id0;
    const int* __restrict__ id1;
    const int* __restrict__ pidx0;  // entry 0's index in the current list (null: via id0)
    // fused force reduction (LBG_FORCE_FUSED)
    const lbg_snapshot* __restrict__ snaps;
    int n_snaps;
    SnapIndex sidx;
    int blk_lo[3];
    double* __restrict__ facc;
    int* __restrict__ fused_used;
    // box launch
    int lo[3], hi[3];
    int i0;  // aligned chunk origin
    // flat launch / list range test
    int nbox;
    int blo[8][3];
    int bext[8][3];
    long long bstart[9];
    int* wc;          // checked build: per-cell write counts
    long long cells;  // interior cells (field length)
};

// checked build: the cell (i, j, k) was written by this sweep
__device__ __forceinline__ void mark_write(const SweepArgs& a, int i, int j, int k) {
#ifdef LBG_CHECKED
    atomicAdd(&a.wc[LBG_IDX(a.L.frac(i, j, k), a.cells, a.err)], 1);
#endif
}

// pull the 19 populations of cell (i,j,k), wrapping periodic axes in-kernel
__device__ __forceinline__ void pull(const SweepArgs& a, int i, int j, int k, long long base,
                                     double (&f)[kQ]) {
    const Layout& L = a.L;
    const long long sy = L.px, sz = (long long)L.px * L.py;
    const long long xl = (a.wrap[0] && i == 0) ? L.nx : 0;  // source i-1 = -1 -> nx-1
    const long long xh = (a.wrap[0] && i == L.nx - 1) ? -(long long)L.nx : 0;
    const long long yl = (a.wrap[1] && j == 0) ? L.ny * sy : 0;
    const long long yh = (a.wrap[1] && j == L.ny - 1) ? -L.ny * sy : 0;
    const long long zl = (a.wrap[2] && k == 0) ? L.nz * sz : 0;
    const long long zh = (a.wrap[2] && k == L.nz - 1) ? -L.nz * sz : 0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const long long corr = (cx(q) == 1 ? xl : (cx(q) == -1 ? xh : 0)) +
                               (cy(q) == 1 ? yl : (cy(q) == -1 ? yh : 0)) +
                               (cz(q) == 1 ? zl : (cz(q) == -1 ? zh : 0));
        f[q] = a.src[q * L.plane + LBG_IDX(base - L.shift(q) + corr, L.plane, a.err)];
    }
}

// PDF loads of the unwrapped pull. A/B builds: -DLBG_LOAD_HINT=1 the streaming load
// (ld.global.cs), =2 no L1 allocation (ld.global.nc.L1::no_allocate)
__device__ __forceinline__ double pdf_load(const double* p) {
#if defined(LBG_LOAD_HINT) && LBG_LOAD_HINT == 1
    return __ldcs(p);
#elif defined(LBG_LOAD_HINT) && LBG_LOAD_HINT == 2
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#else
    return *p;
#endif
}

// pull() for a block with no in-kernel wrap: no per-population wrap selects
template <bool kWrap>
__device__ __forceinline__ void pull_t(const SweepArgs& a, int i, int j, int k, long long base, double (&f)[kQ]) {
    if constexpr (kWrap) {
        pull(a, i, j, k, base, f);
    } else {
        const Layout& L = a.L;
#pragma unroll
        for (int q = 0; q < kQ; ++q) f[q] = pdf_load(a.src + q * L.plane + LBG_IDX(base - L.shift(q), L.plane, a.err));
    }
}

// plain cell; in a coupled block covered cells are left to K2 (kSkipCovered)
template <bool kForced, bool kSkipCovered>
__device__ __forceinline__ bool srt_cell_at(const SweepArgs& a, int i, int j, int k) {
    if constexpr (kSkipCovered) {
        if (a.count[a.L.frac(i, j, k)] != 0) return true;
    }
    const long long base = LBG_IDX(a.L.idx(i, j, k), a.L.plane, a.err);
    double f[kQ];
    pull(a, i, j, k, base, f);
    const bool ok = srt_cell<kForced>(f, a.inv_tau, a.F);
#pragma unroll
    for (int q = 0; q < kQ; ++q) a.dst[q * a.L.plane + base] = f[q];
    mark_write(a, i, j, k);
    return ok;
}

// solid velocity of entry e of cell (i, j, k): with kVsnap, set_solid_velocities' value
// u + cross(omega, c - x) (psm.cpp:157-163, vec3.hpp:39-41; the operations of setu_kernel)
// from the current snapshot list, else the stored field v0/v1
template <bool kVsnap>
__device__ __forceinline__ void solid_velocity(const SweepArgs& a, int e, long long fc, int i, int j, int k,
                                               double (&v)[3]) {
    if constexpr (kVsnap) {
        const int p = a.sidx(e == 0 ? a.id0[fc] : a.id1[fc]);
        if (p < 0) {  // cannot happen for a v_snap field (checked on the host); never read wild
            atomicAdd(&a.err->unknown, 1ull);
            v[0] = v[1] = v[2] = 0.0;
            return;
        }
        const lbg_snapshot& s = a.snaps[p];
        const double r0 = ((double)(a.blk_lo[0] + i) + 0.5) - s.x[0];
        const double r1 = ((double)(a.blk_lo[1] + j) + 0.5) - s.x[1];
        const double r2 = ((double)(a.blk_lo[2] + k) + 0.5) - s.x[2];
        v[0] = s.u[0] + (s.omega[1] * r2 - s.omega[2] * r1);
        v[1] = s.u[1] + (s.omega[2] * r0 - s.omega[0] * r2);
        v[2] = s.u[2] + (s.omega[0] * r1 - s.omega[1] * r0);
    } else {
        const double* w = (e == 0 ? a.v0 : a.v1) + 3 * fc;
        v[0] = w[0];
        v[1] = w[1];
        v[2] = w[2];
    }
}

// snapshot index of entry 0 of cell fc for the inline solid velocity: the mapping's own index
// (a.pidx0, written by the mapping kernel) while the current snapshot list is the mapping list —
// one dependent load instead of id0 -> id table -> index — else snapshot_index(id0)
// (psm.cpp:46-51). For an uncovered cell the value is stale and selected away by the caller.
__device__ __forceinline__ int entry0_index(const SweepArgs& a, long long fc) {
    if (a.pidx0) {
        const int p = a.pidx0[fc];
        return (unsigned)p < (unsigned)a.n_snaps ? p : -1;
    }
    return a.sidx(a.id0[fc]);
}

// solid velocity of an entry named by its particle id (entry 1 of a two-entry cell)
template <bool kVsnap>
__device__ __forceinline__ void solid_velocity_id(const SweepArgs& a, int id, long long fc, int i, int j, int k,
                                                  double (&v)[3]) {
    if constexpr (kVsnap) {
        const int p = a.sidx(id);
        if (p < 0) {
            atomicAdd(&a.err->unknown, 1ull);
            v[0] = v[1] = v[2] = 0.0;
            return;
        }
        const lbg_snapshot& s = a.snaps[p];
        const double r0 = ((double)(a.blk_lo[0] + i) + 0.5) - s.x[0];
        const double r1 = ((double)(a.blk_lo[1] + j) + 0.5) - s.x[1];
        const double r2 = ((double)(a.blk_lo[2] + k) + 0.5) - s.x[2];
        v[0] = s.u[0] + (s.omega[1] * r2 - s.omega[2] * r1);
        v[1] = s.u[1] + (s.omega[2] * r0 - s.omega[0] * r2);
        v[2] = s.u[2] + (s.omega[0] * r1 - s.omega[1] * r0);
    } else {
        const double* w = a.v1 + 3 * fc;
        v[0] = w[0];
        v[1] = w[1];
        v[2] = w[2];
    }
}

// solid velocity of the first entry of a one-entry-segment lane, selected to 0 where the cell
// is not covered. Every index load (id0 or the direct index, the id -> index table, the
// snapshot) is issued without waiting for the cell's count, so the chain seg_list -> cell
// fields -> table -> snapshot overlaps the 19 population loads instead of following them.
// `p` is the entry's snapshot index (kVsnap; -1 if unknown).
template <bool kVsnap>
__device__ __forceinline__ void solid_velocity_sel(const SweepArgs& a, bool cov, long long fc, int i, int j,
                                                   int k, double (&v)[3], int p = -1) {
    if constexpr (kVsnap) {
        if (cov && p < 0) atomicAdd(&a.err->unknown, 1ull);
        double x[3] = {0.0, 0.0, 0.0}, u[3] = {0.0, 0.0, 0.0}, w[3] = {0.0, 0.0, 0.0};
        if (p >= 0) {
            const lbg_snapshot& s = a.snaps[p];
            for (int d = 0; d < 3; ++d) {
                x[d] = s.x[d];
                u[d] = s.u[d];
                w[d] = s.omega[d];
            }
        }
        const double r0 = ((double)(a.blk_lo[0] + i) + 0.5) - x[0];
        const double r1 = ((double)(a.blk_lo[1] + j) + 0.5) - x[1];
        const double r2 = ((double)(a.blk_lo[2] + k) + 0.5) - x[2];
        const bool use = cov && p >= 0;
        v[0] = use ? u[0] + (w[1] * r2 - w[2] * r1) : 0.0;
        v[1] = use ? u[1] + (w[2] * r0 - w[0] * r2) : 0.0;
        v[2] = use ? u[2] + (w[0] * r1 - w[1] * r0) : 0.0;
    } else {
        const double* w = a.v0 + 3 * fc;
        const double w0 = w[0], w1 = w[1], w2 = w[2];
        v[0] = cov ? w0 : 0.0;
        v[1] = cov ? w1 : 0.0;
        v[2] = cov ? w2 : 0.0;
    }
}

__device__ __forceinline__ void count_bad(DeviceErrors* err, bool bad) {
    const unsigned m = __ballot_sync(0xffffffffu, bad);
    if (m && (threadIdx.x & 31) == 0) atomicAdd(&err->unstable, (unsigned long long)__popc(m));
}

template <bool kForced, bool kSkipCovered>
__global__ void __launch_bounds__(256) sweep_box_kernel(const SweepArgs a) {
    const int i = a.i0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int j = a.lo[1] + blockIdx.y * blockDim.y + threadIdx.y;
    const int k = a.lo[2] + blockIdx.z;
    const bool active = i >= a.lo[0] && i < a.hi[0] && j < a.hi[1];
    bool ok = true;
    if constexpr (kSkipCovered) {
        // a warp is one aligned 32-cell row segment; a segment holding any covered cell is
        // swept whole by K2 (psm_seg kernels), so no DRAM sector is touched by both kernels
        const bool cov = i < a.L.nx && j < a.L.ny && a.count[a.L.frac(i, j, k)] != 0;
        if (__any_sync(0xffffffffu, cov)) return;
    }
    if (active) ok = srt_cell_at<kForced, false>(a, i, j, k);
    count_bad(a.err, !ok);
}

// K1 with 128-bit accesses: a lane owns the aligned cell pair (i, i+1), i even, so every
// q-plane is read and written as one double2 per lane (a warp moves 64 cells = four 128-B
// lines per plane). The x-shifted populations come from the neighbour lane's pair by shuffle
// (cx = +1 pulls x-1: lane-1's .y; cx = -1 pulls x+2: lane+1's .x); only the warp's edge lanes
// issue one extra 8-byte load per shifted q. Row j is warp-uniform (blockDim.x = 32).
// Lanes past the box still load their (in-allocation) pair so the shuffles see every lane;
// they store nothing. Cell arithmetic is srt_cell, unchanged, so results are bitwise those of
// the scalar kernel.
template <bool kForced>
__global__ void __launch_bounds__(256, 2) sweep_pair_kernel(const SweepArgs a) {
    const Layout& L = a.L;
    const int lane = threadIdx.x;
    const int i = a.i0 + 2 * (blockIdx.x * 32 + lane);
    const int j = a.lo[1] + blockIdx.y * blockDim.y + threadIdx.y;
    const int k = a.lo[2] + blockIdx.z;
    if (j >= a.hi[1]) return;  // warp-uniform
    const bool actA = i >= a.lo[0] && i < a.hi[0];
    const bool actB = i + 1 >= a.lo[0] && i + 1 < a.hi[0];
    const long long sy = L.px, sz = (long long)L.px * L.py;
    const long long yl = (a.wrap[1] && j == 0) ? L.ny * sy : 0;
    const long long yh = (a.wrap[1] && j == L.ny - 1) ? -L.ny * sy : 0;
    const long long zl = (a.wrap[2] && k == 0) ? L.nz * sz : 0;
    const long long zh = (a.wrap[2] && k == L.nz - 1) ? -L.nz * sz : 0;
    // x positions the edge lanes fetch (x-1 for lane 0, x+2 for lane 31), wrapped if periodic
    const int xm = (a.wrap[0] && i == 0) ? L.nx - 1 : i - 1;
    const int xp = (a.wrap[0] && i + 2 == L.nx) ? 0 : i + 2;
    const long long base = L.idx(i, j, k);
    double fa[kQ], fb[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        // row of the pulled populations: base shifted by -(cy, cz), wrapped per axis
        const long long row = base + q * L.plane - cy(q) * sy - cz(q) * sz +
                              (cy(q) == 1 ? yl : (cy(q) == -1 ? yh : 0)) +
                              (cz(q) == 1 ? zl : (cz(q) == -1 ? zh : 0));
        const double2 v = *reinterpret_cast<const double2*>(a.src + row);
        if (cx(q) == 0) {
            fa[q] = v.x;
            fb[q] = v.y;
        } else if (cx(q) == 1) {
            double e = 0.0;
            if (lane == 0) e = a.src[row - i + xm];
            const double up = __shfl_up_sync(0xffffffffu, v.y, 1);
            fa[q] = lane == 0 ? e : up;
            fb[q] = v.x;
        } else {
            double e = 0.0;
            if (lane == 31) e = a.src[row - i + xp];
            const double dn = __shfl_down_sync(0xffffffffu, v.x, 1);
            fa[q] = v.y;
            fb[q] = lane == 31 ? e : dn;
        }
    }
    if (a.wrap[0]) {
        // the cell at x = nx-1 pulls cx = -1 from x = 0 (unless it sits in lane 31's .y slot,
        // which the edge load already wrapped)
        const bool fixA = i == L.nx - 1, fixB = i + 1 == L.nx - 1 && lane != 31;
        if (fixA || fixB) {
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                if (cx(q) != -1) continue;
                const long long row = base + q * L.plane - cy(q) * sy - cz(q) * sz +
                                      (cy(q) == 1 ? yl : (cy(q) == -1 ? yh : 0)) +
                                      (cz(q) == 1 ? zl : (cz(q) == -1 ? zh : 0));
                const double w = a.src[row - i];  // x = 0
                if (fixA) fa[q] = w;
                if (fixB) fb[q] = w;
            }
        }
    }
    const bool okA = srt_cell<kForced>(fa, a.inv_tau, a.F);
    const bool okB = srt_cell<kForced>(fb, a.inv_tau, a.F);
    double* d = a.dst + LBG_IDX(base, L.plane, a.err);
    if (actA) mark_write(a, i, j, k);
    if (actB) mark_write(a, i + 1, j, k);
    if (actA && actB) {
#pragma unroll
        for (int q = 0; q < kQ; ++q)
            *reinterpret_cast<double2*>(d + q * L.plane) = make_double2(fa[q], fb[q]);
    } else if (actA || actB) {
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            if (actA) d[q * L.plane] = fa[q];
            if (actB) d[q * L.plane + 1] = fb[q];
        }
    }
    const unsigned ma = __ballot_sync(0xffffffffu, actA && !okA);
    const unsigned mb = __ballot_sync(0xffffffffu, actB && !okB);
    if ((ma | mb) && lane == 0) atomicAdd(&a.err->unstable, (unsigned long long)(__popc(ma) + __popc(mb)));
}

__device__ __forceinline__ void flat_cell(const SweepArgs& a, long long t, int& i, int& j, int& k) {
    int b = 0;
    while (t >= a.bstart[b + 1]) ++b;
    const long long r = t - a.bstart[b];
    const int ex = a.bext[b][0], ey = a.bext[b][1];
    i = a.blo[b][0] + (int)(r % ex);
    j = a.blo[b][1] + (int)((r / ex) % ey);
    k = a.blo[b][2] + (int)(r / ((long long)ex * ey));
}

template <bool kForced, bool kSkipCovered>
__global__ void __launch_bounds__(256) sweep_flat_kernel(const SweepArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (t < a.bstart[a.nbox]) {
        int i, j, k;
        flat_cell(a, t, i, j, k);
        ok = srt_cell_at<kForced, kSkipCovered>(a, i, j, k);
    }
    count_bad(a.err, !ok);
}

__device__ __forceinline__ bool in_boxes(const SweepArgs& a, int i, int j, int k) {
    for (int b = 0; b < a.nbox; ++b)
        if (i >= a.blo[b][0] && i < a.blo[b][0] + a.bext[b][0] && j >= a.blo[b][1] &&
            j < a.blo[b][1] + a.bext[b][1] && k >= a.blo[b][2] && k < a.blo[b][2] + a.bext[b][2])
            return true;
    return false;
}

// LBG_FORCE_FUSED: lanes holding an entry of the same particle form a group (match_any);
// the group leader sums the group's force and torque (cross(c - x_p, m), psm.cpp:296) by
// shuffles in lane order and issues one atomicAdd per component.
__device__ __forceinline__ void fused_accumulate(const SweepArgs& a, int p, const double (&m)[3],
                                                 const double (&cc)[3]) {
    double v[6] = {0, 0, 0, 0, 0, 0};
    if (p >= 0) {
        const lbg_snapshot& s = a.snaps[p];
        const double r0 = cc[0] - s.x[0], r1 = cc[1] - s.x[1], r2 = cc[2] - s.x[2];
        v[0] = m[0];
        v[1] = m[1];
        v[2] = m[2];
        v[3] = r1 * m[2] - r2 * m[1];
        v[4] = r2 * m[0] - r0 * m[2];
        v[5] = r0 * m[1] - r1 * m[0];
    }
    const unsigned peers = __match_any_sync(0xffffffffu, p);
    if (p < 0) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    double s[6] = {0, 0, 0, 0, 0, 0};
    unsigned rest = peers;
    while (rest) {
        const int src = __ffs(rest) - 1;
        rest &= rest - 1;
#pragma unroll
        for (int d = 0; d < 6; ++d) s[d] += __shfl_sync(peers, v[d], src);
    }
    if (lane == leader) {
#pragma unroll
        for (int d = 0; d < 6; ++d) atomicAdd(&a.facc[6 * p + d], s[d]);
        a.fused_used[p] = 1;
    }
}

// One lane of the coupled sweep at interior cell (i, j, k) with fraction count cnt: SRT
// (count 0), the pair-scheduled one-entry operator (count 1) or, with kGeneral, the general
// operator (count 2). For the fused force mode it also names the entries' particles (p0, p1)
// and the cell centre for fused_accumulate.
template <bool kForced, bool kFused, bool kGeneral, bool kVsnap>
__device__ __forceinline__ bool coupled_lane(const SweepArgs& a, int i, int j, int k, long long fc, int cnt,
                                             double (&m)[2][3], int& p0, int& p1, double (&cc)[3]) {
    const Layout& L = a.L;
    fc = LBG_IDX(fc, a.cells, a.err);
    (void)LBG_IDX(L.idx(i, j, k), L.plane, a.err);
    bool ok;
    if (!kGeneral && !kForced) {
        // unforced one-entry lanes: fluid lanes run the same operator with B = b = 0 and
        // v = 0, which is collide_cell exactly (fluid weight 1 - 0 = 1, f + 1 * coll ==
        // f + coll, and the solid term adds 0 * C = +-0 to a nonzero value), so a mixed warp
        // issues one operator instead of SRT and PSM in turn
        const bool cov = cnt > 0;
        const long long base = L.idx(i, j, k);
        // cell fields loaded unconditionally (fc is an interior cell), selected by cov
        const double bt = a.btot[fc], b0 = a.b0[fc];
        double v[3];
        const int pe = kVsnap ? entry0_index(a, fc) : -1;
        solid_velocity_sel<kVsnap>(a, cov, fc, i, j, k, v, pe);
        double f[kQ];
        pull(a, i, j, k, base, f);
        ok = psm_cell_one<kForced>(f, a.inv_tau, a.F, cov ? bt : 0.0, cov ? b0 : 0.0, v[0], v[1], v[2], a.dst,
                                   L.plane, base, m[0]);
        if constexpr (!kFused)
            if (cov)
                for (int d = 0; d < 3; ++d) a.m0[3 * fc + d] = m[0][d];
    } else if (!kGeneral && cnt == 0) {
        ok = srt_cell_at<kForced, false>(a, i, j, k);
    } else if constexpr (!kGeneral) {
        const long long base = L.idx(i, j, k);
        double f[kQ];
        pull(a, i, j, k, base, f);
        double v[3];
        solid_velocity<kVsnap>(a, 0, fc, i, j, k, v);
        ok = psm_cell_one<kForced>(f, a.inv_tau, a.F, a.btot[fc], a.b0[fc], v[0], v[1], v[2], a.dst, L.plane,
                                   base, m[0]);
        if constexpr (!kFused)
            for (int d = 0; d < 3; ++d) a.m0[3 * fc + d] = m[0][d];
    } else if (!kForced || cnt > 0) {
        // two-entry segments: the pair-scheduled operator with entry 1 where cnt > 1 (unforced
        // fluid lanes as in the one-entry case: B = b = 0, v = 0)
        const bool cov = cnt > 0, two = cnt > 1;
        const long long base = L.idx(i, j, k);
        const double bt = a.btot[fc], b0 = a.b0[fc], b1 = a.b1[fc];
        double v0[3], v1[3] = {0.0, 0.0, 0.0};
        const int pe = kVsnap ? entry0_index(a, fc) : -1;
        solid_velocity_sel<kVsnap>(a, cov, fc, i, j, k, v0, pe);
        if (two) solid_velocity<kVsnap>(a, 1, fc, i, j, k, v1);
        double f[kQ];
        pull(a, i, j, k, base, f);
        ok = psm_cell_two<kForced>(f, a.inv_tau, a.F, cov ? bt : 0.0, cov ? b0 : 0.0, v0, two ? b1 : 0.0, v1, two,
                                   a.dst, L.plane, base, m);
        if constexpr (!kFused) {
            if (cov)
                for (int d = 0; d < 3; ++d) a.m0[3 * fc + d] = m[0][d];
            if (two)
                for (int d = 0; d < 3; ++d) a.m1[3 * fc + d] = m[1][d];
        }
    } else {
        ok = srt_cell_at<kForced, false>(a, i, j, k);
    }
    // the psm branches store through the pair operators: count their cell here (the forced
    // fluid lanes went through srt_cell_at, which counts its own)
    if (!(kForced && cnt == 0)) mark_write(a, i, j, k);
    if constexpr (kFused) {
        if (cnt > 0) {
            cc[0] = (double)(a.blk_lo[0] + i) + 0.5;
            cc[1] = (double)(a.blk_lo[1] + j) + 0.5;
            cc[2] = (double)(a.blk_lo[2] + k) + 0.5;
            p0 = entry0_index(a, fc);
            if (cnt > 1) p1 = a.sidx(a.id1[fc]);
            if (p0 < 0 || (cnt > 1 && p1 < 0)) atomicAdd(&a.err->unknown, 1ull);
        }
    }
    return ok;
}

// K2: one warp per covered 32-cell row segment (segment lists written by the mapping kernel).
// Each lane takes its cell through SRT (count 0), the pair-scheduled one-entry operator
// (count 1) or — in segments holding a two-entry cell (kTwo) — the general operator. K1 skips
// exactly these segments, so every DRAM sector of the PDF planes is read and written once.
template <bool kForced, bool kFused, bool kTwo, bool kVsnap>
__global__ void __launch_bounds__(128) psm_seg_kernel(const SweepArgs a) {
    const int nseg = kTwo ? a.seg_n[1] : a.seg_n[0];
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    const Layout& L = a.L;
    auto seg_at = [&](int s) { return kTwo ? a.seg_list[a.seg_cap - 1 - s] : a.seg_list[s]; };
    unsigned c_next = warp < nseg ? seg_at(warp) : 0u;
    for (int s = warp; s < nseg; s += nwarps) {
        const unsigned c0 = c_next;
        if (s + nwarps < nseg) c_next = seg_at(s + nwarps);  // the next segment's origin in flight
        const int i = (int)(c0 % (unsigned)L.nx) + lane;
        const int j = (int)((c0 / (unsigned)L.nx) % (unsigned)L.ny);
        const int k = (int)(c0 / ((unsigned)L.nx * (unsigned)L.ny));
        bool ok = true;
        double m[2][3] = {{0, 0, 0}, {0, 0, 0}};
        double cc[3] = {0, 0, 0};
        int p0 = -1, p1 = -1;
        if (i < L.nx && in_boxes(a, i, j, k)) {
            const long long fc = L.frac(i, j, k);
            ok = coupled_lane<kForced, kFused, kTwo, kVsnap>(a, i, j, k, fc, a.count[fc], m, p0, p1, cc);
        }
        count_bad(a.err, !ok);
        if constexpr (kFused) {
            fused_accumulate(a, p0, m[0], cc);
            fused_accumulate(a, p1, m[1], cc);
        }
    }
}

// K2 for unforced one-entry segments with software pipelining across the grid-stride loop:
// the next segment's populations and cell fields are loaded (SegIn) before the current
// segment's arithmetic, so a warp's DRAM latency hides behind its own fp64 work instead of
// only behind other warps'. Same per-lane operator as psm_seg_kernel<false, *, false, *>.
struct SegIn {
    double f[kQ];
    double bt, b0;
    long long fc, base;
    int i, j, k, cnt, id0;
    bool act;
};

template <bool kVsnap>
__device__ __forceinline__ void seg_load(const SweepArgs& a, unsigned c0, int lane, SegIn& in) {
    const Layout& L = a.L;
    in.i = (int)(c0 % (unsigned)L.nx) + lane;
    in.j = (int)((c0 / (unsigned)L.nx) % (unsigned)L.ny);
    in.k = (int)(c0 / ((unsigned)L.nx * (unsigned)L.ny));
    in.act = in.i < L.nx && in_boxes(a, in.i, in.j, in.k);
    in.cnt = 0;
    if (in.act) {
        in.fc = LBG_IDX(L.frac(in.i, in.j, in.k), a.cells, a.err);
        in.base = LBG_IDX(L.idx(in.i, in.j, in.k), L.plane, a.err);
        in.cnt = a.count[in.fc];
        in.bt = a.btot[in.fc];
        in.b0 = a.b0[in.fc];
        if constexpr (kVsnap) in.id0 = a.id0[in.fc];
        pull(a, in.i, in.j, in.k, in.base, in.f);
    }
}

// first half of a segment's update: everything that consumes the segment's loaded registers
// (solid velocity from its id, the moments). The pipelined loop issues the next segment's
// loads only after this, so no wait on this segment's data can also wait on those loads
// (loads share the warp's few scoreboard counters).
struct SegPre {
    double v[3];
    double rho, ux, uy, uz, usq;
    bool ok;
};

template <bool kVsnap>
__device__ __forceinline__ void seg_pre(const SweepArgs& a, const SegIn& in, SegPre& pre) {
    if (!in.act) return;
    solid_velocity_sel<kVsnap>(a, in.cnt > 0, in.fc, in.i, in.j, in.k, pre.v, kVsnap ? a.sidx(in.id0) : -1);
    moments(in.f, pre.rho, pre.ux, pre.uy, pre.uz);
    pre.usq = (pre.ux * pre.ux + pre.uy * pre.uy) + pre.uz * pre.uz;
    pre.ok = pre.rho > 0.0 && pre.usq <= kMaxVelocity * kMaxVelocity && isfinite(pre.rho);
}

template <bool kFused, bool kVsnap>
__device__ __forceinline__ void seg_finish(const SweepArgs& a, const SegIn& in, const SegPre& pre) {
    bool ok = true;
    double m[3] = {0, 0, 0};
    double cc[3] = {0, 0, 0};
    int p0 = -1;
    if (in.act) {
        const bool cov = in.cnt > 0;
        psm_cell_one_pairs<false>(in.f, pre.rho, pre.ux, pre.uy, pre.uz, pre.usq, a.inv_tau, a.F,
                                  cov ? in.bt : 0.0, cov ? in.b0 : 0.0, pre.v[0], pre.v[1], pre.v[2], a.dst,
                                  a.L.plane, in.base, m);
        ok = pre.ok;
        mark_write(a, in.i, in.j, in.k);
        if constexpr (!kFused) {
            if (cov)
                for (int d = 0; d < 3; ++d) a.m0[3 * in.fc + d] = m[d];
        } else if (cov) {
            cc[0] = (double)(a.blk_lo[0] + in.i) + 0.5;
            cc[1] = (double)(a.blk_lo[1] + in.j) + 0.5;
            cc[2] = (double)(a.blk_lo[2] + in.k) + 0.5;
            p0 = a.sidx(kVsnap ? in.id0 : a.id0[in.fc]);
            if (p0 < 0) atomicAdd(&a.err->unknown, 1ull);
        }
    }
    count_bad(a.err, !ok);
    if constexpr (kFused) fused_accumulate(a, p0, m, cc);
}

template <bool kFused, bool kVsnap>
__global__ void __launch_bounds__(128) psm_seg_pipe_kernel(const SweepArgs a) {
    const int nseg = a.seg_n[0];
    const int lane = threadIdx.x & 31;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    if (warp >= nseg) return;  // warp-uniform
    SegIn cur, nxt;
    SegPre pre;
    seg_load<kVsnap>(a, a.seg_list[warp], lane, cur);
    int s = warp;
    for (;;) {
        const bool more = s + nwarps < nseg;
        seg_pre<kVsnap>(a, cur, pre);
        if (more) seg_load<kVsnap>(a, a.seg_list[s + nwarps], lane, nxt);
        seg_finish<kFused, kVsnap>(a, cur, pre);
        if (!more) break;
        s += nwarps;
        // second half of the unrolled pair: roles swapped, no register copy
        const bool more2 = s + nwarps < nseg;
        seg_pre<kVsnap>(a, nxt, pre);
        if (more2) seg_load<kVsnap>(a, a.seg_list[s + nwarps], lane, cur);
        seg_finish<kFused, kVsnap>(a, nxt, pre);
        if (!more2) break;
        s += nwarps;
    }
}

// K2 for unforced one-entry segments fed by the Tensor Memory Accelerator: per warp, lane 0
// issues one 1-D bulk copy (cp.async.bulk, completion counted on an mbarrier) per pulled
// q-row — the 40 doubles [i0 - 4, i0 + 36) of the row the direction pulls from, with the
// periodic y/z wrap applied to the row — plus the segment's btot, b0, id0 and count
// windows, into one of two shared-memory stages, while the warp computes the previous
// segment from the other stage. A lane's population q is stage.f[q][4 + lane - c_x(q)].
// 23 copy instructions per segment instead of 23 loads per lane, and nothing in flight
// occupies registers or the warp's scoreboards (the register-pipelined variant stalled on
// them; per-lane cp.async saturated the LSU queue: profiles/r01_ab_k2.txt). Lanes at an
// x-wrapped block face re-pull from global (pull()).
struct SegStage {
    double f[kQ][40];
    double bt[34];
    double b0[34];
    int id0[36];
    unsigned char cnt[48];
};
static_assert(sizeof(SegStage) % 16 == 0, "stage must keep 16-byte alignment");
constexpr int kTmaWarps = 4;  // warps per CTA (128 threads), two stages each
constexpr unsigned kRowBytes = 40 * 8;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    unsigned done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// lane 0: the copies of segment c0 into `st`, completing on `bar`
template <bool kVsnap>
__device__ __forceinline__ void seg_tma_issue(const SweepArgs& a, unsigned c0, SegStage& st,
                                              unsigned long long* bar) {
    const Layout& L = a.L;
    const int i0 = (int)(c0 % (unsigned)L.nx);
    const int j = (int)((c0 / (unsigned)L.nx) % (unsigned)L.ny);
    const int k = (int)(c0 / ((unsigned)L.nx * (unsigned)L.ny));
    const unsigned tx = kQ * kRowBytes + 2 * 272 + (kVsnap ? 144 : 0) + 48;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of st
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
    const long long sy = L.px, sz = (long long)L.px * L.py;
    const long long yl = (a.wrap[1] && j == 0) ? L.ny * sy : 0;
    const long long yh = (a.wrap[1] && j == L.ny - 1) ? -L.ny * sy : 0;
    const long long zl = (a.wrap[2] && k == 0) ? L.nz * sz : 0;
    const long long zh = (a.wrap[2] && k == L.nz - 1) ? -L.nz * sz : 0;
    const long long row0 = L.idx(i0, j, k) - 4;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const long long r = q * L.plane + row0 - cy(q) * sy - cz(q) * sz + (cy(q) == 1 ? yl : (cy(q) == -1 ? yh : 0)) +
                            (cz(q) == 1 ? zl : (cz(q) == -1 ? zh : 0));
        tma_bulk(st.f[q], a.src + r, kRowBytes, bar);
    }
    const long long c = (long long)c0;
    tma_bulk(st.bt, a.btot + (c & ~1LL), 272, bar);
    tma_bulk(st.b0, a.b0 + (c & ~1LL), 272, bar);
    if constexpr (kVsnap) tma_bulk(st.id0, a.id0 + (c & ~3LL), 144, bar);
    tma_bulk(st.cnt, a.count + (c & ~15LL), 48, bar);
}

template <bool kFused, bool kVsnap>
__device__ __forceinline__ void seg_from_tma(const SweepArgs& a, unsigned c0, int lane, const SegStage& st) {
    const Layout& L = a.L;
    const int i = (int)(c0 % (unsigned)L.nx) + lane;
    const int j = (int)((c0 / (unsigned)L.nx) % (unsigned)L.ny);
    const int k = (int)(c0 / ((unsigned)L.nx * (unsigned)L.ny));
    const bool act = i < L.nx && in_boxes(a, i, j, k);
    bool ok = true;
    double m[3] = {0, 0, 0};
    double cc[3] = {0, 0, 0};
    int p0 = -1;
    if (act) {
        const long long base = LBG_IDX(L.idx(i, j, k), L.plane, a.err), fc = LBG_IDX(L.frac(i, j, k), a.cells, a.err);
        mark_write(a, i, j, k);
        const int cnt = st.cnt[lane + (int)(c0 & 15u)];
        const bool cov = cnt > 0;
        const int id0 = kVsnap ? st.id0[lane + (int)(c0 & 3u)] : 0;
        const double bt = st.bt[lane + (int)(c0 & 1u)], b0 = st.b0[lane + (int)(c0 & 1u)];
        double f[kQ];
        if (a.wrap[0] && (i == 0 || i == L.nx - 1)) {
            pull(a, i, j, k, base, f);
        } else {
#pragma unroll
            for (int q = 0; q < kQ; ++q) f[q] = st.f[q][4 + lane - cx(q)];
        }
        double v[3];
        solid_velocity_sel<kVsnap>(a, cov, fc, i, j, k, v, kVsnap ? a.sidx(id0) : -1);
        ok = psm_cell_one<false>(f, a.inv_tau, a.F, cov ? bt : 0.0, cov ? b0 : 0.0, v[0], v[1], v[2], a.dst,
                                 L.plane, base, m);
        if constexpr (!kFused) {
            if (cov)
                for (int d = 0; d < 3; ++d) a.m0[3 * fc + d] = m[d];
        } else if (cov) {
            cc[0] = (double)(a.blk_lo[0] + i) + 0.5;
            cc[1] = (double)(a.blk_lo[1] + j) + 0.5;
            cc[2] = (double)(a.blk_lo[2] + k) + 0.5;
            p0 = a.sidx(kVsnap ? id0 : a.id0[fc]);
            if (p0 < 0) atomicAdd(&a.err->unknown, 1ull);
        }
    }
    count_bad(a.err, !ok);
    if constexpr (kFused) fused_accumulate(a, p0, m, cc);
}

template <bool kFused, bool kVsnap>
__global__ void __launch_bounds__(32 * kTmaWarps) psm_seg_tma_kernel(const SweepArgs a) {
    extern __shared__ __align__(128) unsigned char seg_smem[];
    const int nseg = a.seg_n[0];
    const int lane = threadIdx.x & 31;
    const int wl = threadIdx.x >> 5;
    const int warp = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    SegStage* stage = reinterpret_cast<SegStage*>(seg_smem) + 2 * wl;
    unsigned long long* bar =
        reinterpret_cast<unsigned long long*>(seg_smem + sizeof(SegStage) * 2 * kTmaWarps) + 2 * wl;
    if (warp >= nseg) return;  // warp-uniform
    if (lane == 0) {
        for (int t = 0; t < 2; ++t)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[t])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    unsigned c_cur = a.seg_list[warp];
    if (lane == 0) seg_tma_issue<kVsnap>(a, c_cur, stage[0], &bar[0]);
    unsigned phase[2] = {0u, 0u};
    int b = 0;
    for (int s = warp; s < nseg; s += nwarps) {
        const bool more = s + nwarps < nseg;
        const unsigned c_next = more ? a.seg_list[s + nwarps] : 0u;
        if (more && lane == 0) seg_tma_issue<kVsnap>(a, c_next, stage[b ^ 1], &bar[b ^ 1]);
        mbar_wait(&bar[b], phase[b]);
        phase[b] ^= 1u;
        seg_from_tma<kFused, kVsnap>(a, c_cur, lane, stage[b]);
        __syncwarp();  // every lane is done with stage b before lane 0 refills it
        c_cur = c_next;
        b ^= 1;
    }
}

// ---------------------------------------------------------------- K12: unified coupled sweep
// One persistent kernel for the fluid and the one-entry segments of a coupled block (default;
// LBG_K12=0 restores the K1 || K2 split): each warp walks the aligned 32-cell row segments of
// the box in memory order (grid stride), reads the segment's 32 count bytes and runs the SRT
// operator (no covered cell) or the pair-scheduled one-entry operator on every lane (max count
// 1; fluid lanes with B = b = 0 when unforced). Segments holding a two-entry cell are left to
// psm_seg_kernel<two> (the segment list's back), so every PDF sector is still swept by exactly
// one kernel. One kernel keeps the SM's warps mixing memory-bound SRT segments with the
// fp64-heavy PSM segments (the split had early-exit K1 warps and, the register file being
// full with K2, no real K1 || K2 concurrency). Config 3: 1.09 ms vs 1.13 ms for the split
// (profiles/r02_ab_k12.txt, where the variants that measured slower are listed: L2 bulk or
// line prefetch of the next segment, a dynamic segment counter, a low-register L1-re-read
// operator, 4 or 6 CTAs per SM).
template <bool kForced, bool kFused, bool kVsnap, int kMinBlocks>
__global__ void __launch_bounds__(128, kMinBlocks) coupled_unified_kernel(const SweepArgs a) {
    const Layout& L = a.L;
    const int lane = threadIdx.x & 31;
    const long long warp = (long long)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const long long nwarps = (long long)((gridDim.x * blockDim.x) >> 5);
    const int segs_x = (a.hi[0] - a.i0 + 31) >> 5;
    const int ny_b = a.hi[1] - a.lo[1];
    const long long nseg = (long long)segs_x * ny_b * (a.hi[2] - a.lo[2]);
    if (warp >= nseg) return;  // warp-uniform
    // the count byte of a segment is loaded one segment ahead, so the operator choice never
    // waits on HBM and every segment's loads (populations, cell fields) go out in one batch
    auto count_of = [&](long long s) -> int {
        if (s >= nseg) return 0;
        // 32-bit index math (a 64-bit division is a ~100-instruction software routine)
        const unsigned su = (unsigned)s, r = su / (unsigned)segs_x;
        const int i = a.i0 + 32 * (int)(su - r * (unsigned)segs_x) + lane;
        if (i >= L.nx) return 0;
        return (int)a.count[LBG_IDX(L.frac(i, a.lo[1] + (int)(r % (unsigned)ny_b), a.lo[2] + (int)(r / (unsigned)ny_b)),
                                    a.cells, a.err)];
    };
    auto sweep_seg = [&](long long s, int cnt) {
        const unsigned su = (unsigned)s, r = su / (unsigned)segs_x;
        const int i = a.i0 + 32 * (int)(su - r * (unsigned)segs_x) + lane;
        const int j = a.lo[1] + (int)(r % (unsigned)ny_b);
        const int k = a.lo[2] + (int)(r / (unsigned)ny_b);
        const int mx = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
        if (mx >= 2) return;  // psm_seg_kernel<two> sweeps this segment
        const bool act = i < L.nx && i >= a.lo[0] && i < a.hi[0];
        bool ok = true;
        if (mx == 0) {
            if (act) ok = srt_cell_at<kForced, false>(a, i, j, k);
            count_bad(a.err, !ok);
            return;
        }
        double m[2][3] = {{0, 0, 0}, {0, 0, 0}};
        double cc[3] = {0, 0, 0};
        int p0 = -1, p1 = -1;
        if (act) ok = coupled_lane<kForced, kFused, false, kVsnap>(a, i, j, k, L.frac(i, j, k), cnt, m, p0, p1, cc);
        count_bad(a.err, !ok);
        if constexpr (kFused) fused_accumulate(a, p0, m[0], cc);
    };
    // one body (a second inlined copy of both operators overflows the instruction cache): the
    // copy of the count loaded a whole segment earlier never waits
    int cnt_next = count_of(warp);
    for (long long s = warp; s < nseg; s += nwarps) {
        const int cnt = cnt_next;
        cnt_next = count_of(s + nwarps);
        sweep_seg(s, cnt);
    }
}

// K12, register-pipelined (default; LBG_K12_PIPE=0 selects the plain loop above; unforced,
// inline solid velocities through the mapping's direct index): the next segment's
// populations and cell fields (count, btot, b0, entry index: all loaded, the operator is only
// known when the count arrives) are loaded while the
// current one is finished. pre() consumes everything the current segment loaded (count ballot,
// moments, solid velocity) before the next loads are issued, so no wait on the current data is
// also a wait on the next (loads share the warp's scoreboards); the register sets swap roles
// through the unrolled loop (a copy of an in-flight register would wait for it).
struct USeg {
    double f[kQ];
    double bt, b0, b1;
    long long fc, base;
    int i, j, k, cnt, pe, id1, mx;
    bool act;
};

struct UPre {
    double rho, ux, uy, uz, usq, v[3], v1[3];
    bool ok;
};

// segment s's first cell: dense mode — the s-th aligned 32-cell row segment of the box; list
// mode (kList) — the s-th entry of the mapping's covered-segment list (one-entry segments from
// the front, segments with a two-entry cell from the back)
struct USegId {
    int i0, j, k;
};

// list mode: the list entry of segment s (its first cell index)
__device__ __forceinline__ unsigned useg_raw(const SweepArgs& a, long long s, long long nseg, int n1) {
    if (s >= nseg) return 0u;
    return (s < n1) ? a.seg_list[s] : a.seg_list[a.seg_cap - 1 - (s - n1)];
}

__device__ __forceinline__ USegId useg_decode(const Layout& L, unsigned c0) {
    USegId id;
    const unsigned row = c0 / (unsigned)L.nx;
    id.i0 = (int)(c0 - row * (unsigned)L.nx);
    id.j = (int)(row % (unsigned)L.ny);
    id.k = (int)(row / (unsigned)L.ny);
    return id;
}

__device__ __forceinline__ USegId useg_dense(const SweepArgs& a, long long s, int segs_x, int ny_b) {
    // 32-bit index math (a 64-bit division is a ~100-instruction software routine)
    USegId id;
    const unsigned su = (unsigned)s, r = su / (unsigned)segs_x;
    id.i0 = a.i0 + 32 * (int)(su - r * (unsigned)segs_x);
    id.j = a.lo[1] + (int)(r % (unsigned)ny_b);
    id.k = a.lo[2] + (int)(r / (unsigned)ny_b);
    return id;
}

// the count bytes of segment `id` (32 lanes)
__device__ __forceinline__ int useg_count(const SweepArgs& a, const USegId& id, bool valid, int lane) {
    const Layout& L = a.L;
    const int i = id.i0 + lane;
    if (!valid || i >= L.nx) return 0;
    return (int)a.count[LBG_IDX(L.frac(i, id.j, id.k), a.cells, a.err)];
}

// the loads of segment `id`, whose counts `cnt` arrived one segment earlier: the populations
// unless it is a two-entry segment swept elsewhere, the cell fields only for a covered
// segment — nothing an SRT segment does not use
template <bool kTwoInline, bool kWrap>
__device__ __forceinline__ void useg_issue(const SweepArgs& a, const USegId& id, int lane, int cnt, USeg& u) {
    const Layout& L = a.L;
    u.i = id.i0 + lane;
    u.j = id.j;
    u.k = id.k;
    const bool inx = u.i < L.nx;
    u.fc = LBG_IDX(L.frac(inx ? u.i : L.nx - 1, u.j, u.k), a.cells, a.err);
    u.act = inx && u.i >= a.lo[0] && u.i < a.hi[0] && u.j >= a.lo[1] && u.j < a.hi[1] && u.k >= a.lo[2] &&
            u.k < a.hi[2];
    u.cnt = cnt;
    u.mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
    if (u.mx >= 1) {
        u.bt = a.btot[u.fc];
        u.b0 = a.b0[u.fc];
        u.pe = a.pidx0[u.fc];
    }
    if (kTwoInline && u.mx >= 2) {
        u.b1 = a.b1[u.fc];
        u.id1 = a.id1[u.fc];
    }
    if (u.act && (kTwoInline || u.mx <= 1)) {
        u.base = LBG_IDX(L.idx(u.i, u.j, u.k), L.plane, a.err);
        pull_t<kWrap>(a, u.i, u.j, u.k, u.base, u.f);
    }
}

template <bool kVsnap, bool kTwoInline>
__device__ __forceinline__ void useg_pre(const SweepArgs& a, const USeg& u, UPre& pre) {
    pre.ok = true;
    if ((!kTwoInline && u.mx >= 2) || !u.act) return;
    const bool cov = u.cnt > 0;
    if (u.mx >= 1) {
        const int p = kVsnap ? ((unsigned)u.pe < (unsigned)a.n_snaps ? u.pe : -1) : -1;
        solid_velocity_sel<kVsnap>(a, cov, u.fc, u.i, u.j, u.k, pre.v, p);
    }
    if (kTwoInline && u.mx >= 2) {
        pre.v1[0] = pre.v1[1] = pre.v1[2] = 0.0;
        if (u.cnt > 1) solid_velocity_id<kVsnap>(a, u.id1, u.fc, u.i, u.j, u.k, pre.v1);
    }
    moments(u.f, pre.rho, pre.ux, pre.uy, pre.uz);
    pre.usq = (pre.ux * pre.ux + pre.uy * pre.uy) + pre.uz * pre.uz;
    pre.ok = pre.rho > 0.0 && pre.usq <= kMaxVelocity * kMaxVelocity && isfinite(pre.rho);
}

template <bool kFused, bool kVsnap, bool kTwoInline>
__device__ __forceinline__ void useg_finish(const SweepArgs& a, const USeg& u, const UPre& pre) {
    if (!kTwoInline && u.mx >= 2) return;  // psm_seg_kernel<two> sweeps this segment
    if (kTwoInline && u.mx >= 2) {
        // two-entry segment: the pair-scheduled two-entry operator (entry 1 where count 2)
        double m2[2][3] = {{0, 0, 0}, {0, 0, 0}};
        double cc[3] = {0, 0, 0};
        int p0 = -1, p1 = -1;
        bool ok = true;
        if (u.act) {
            const bool cov = u.cnt > 0, two = u.cnt > 1;
            ok = psm_cell_two<false>(u.f, a.inv_tau, a.F, cov ? u.bt : 0.0, cov ? u.b0 : 0.0, pre.v, two ? u.b1 : 0.0,
                                     pre.v1, two, a.dst, a.L.plane, u.base, m2);
            if constexpr (!kFused) {
                if (cov)
                    for (int d = 0; d < 3; ++d) a.m0[3 * u.fc + d] = m2[0][d];
                if (two)
                    for (int d = 0; d < 3; ++d) a.m1[3 * u.fc + d] = m2[1][d];
            } else if (cov) {
                cc[0] = (double)(a.blk_lo[0] + u.i) + 0.5;
                cc[1] = (double)(a.blk_lo[1] + u.j) + 0.5;
                cc[2] = (double)(a.blk_lo[2] + u.k) + 0.5;
                p0 = (unsigned)u.pe < (unsigned)a.n_snaps ? u.pe : -1;
                if (two) p1 = a.sidx(u.id1);
                if (p0 < 0 || (two && p1 < 0)) atomicAdd(&a.err->unknown, 1ull);
            }
            mark_write(a, u.i, u.j, u.k);
        }
        count_bad(a.err, !ok);
        if constexpr (kFused) {
            fused_accumulate(a, p0, m2[0], cc);
            fused_accumulate(a, p1, m2[1], cc);
        }
        return;
    }
    double m[3] = {0, 0, 0};
    double cc[3] = {0, 0, 0};
    int p0 = -1;
    if (u.act) {
        const auto g = [&](int q) { return u.f[q]; };
        if (u.mx == 0) {
            srt_pairs_g(g, pre.rho, pre.ux, pre.uy, pre.uz, pre.usq, a.inv_tau, a.dst, a.L.plane, u.base);
        } else {
            const bool cov = u.cnt > 0;
            psm_one_pairs_g<false>(g, pre.rho, pre.ux, pre.uy, pre.uz, pre.usq, a.inv_tau, a.F, cov ? u.bt : 0.0,
                                   cov ? u.b0 : 0.0, pre.v[0], pre.v[1], pre.v[2], a.dst, a.L.plane, u.base, m);
            if constexpr (!kFused) {
                if (cov)
                    for (int d = 0; d < 3; ++d) a.m0[3 * u.fc + d] = m[d];
            } else if (cov) {
                cc[0] = (double)(a.blk_lo[0] + u.i) + 0.5;
                cc[1] = (double)(a.blk_lo[1] + u.j) + 0.5;
                cc[2] = (double)(a.blk_lo[2] + u.k) + 0.5;
                p0 = (unsigned)u.pe < (unsigned)a.n_snaps ? u.pe : -1;
                if (p0 < 0) atomicAdd(&a.err->unknown, 1ull);
            }
        }
        mark_write(a, u.i, u.j, u.k);
    }
    count_bad(a.err, !pre.ok);
    if constexpr (kFused)
        if (u.mx == 1) fused_accumulate(a, p0, m, cc);
}

#ifndef LBG_K12_MINB
#define LBG_K12_MINB 3  // CTAs per SM the register budget is set for (A/B builds: 4)
#endif
template <bool kFused, bool kVsnap, bool kTwoInline, bool kWrap, bool kList = false>
__global__ void __launch_bounds__(128, LBG_K12_MINB) coupled_unified_pipe_kernel(const SweepArgs a) {
    const int lane = threadIdx.x & 31;
    const long long warp = (long long)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const long long nwarps = (long long)((gridDim.x * blockDim.x) >> 5);
    const int segs_x = (a.hi[0] - a.i0 + 31) >> 5;
    const int ny_b = a.hi[1] - a.lo[1];
    const int n1 = kList ? a.seg_n[0] : 0;
    const long long nseg = kList ? (long long)n1 + a.seg_n[1] : (long long)segs_x * ny_b * (a.hi[2] - a.lo[2]);
    if (warp >= nseg) return;  // warp-uniform
    // list mode: list entries three segments ahead, decoded when their counts are loaded
    auto locate = [&](long long s, unsigned raw) {
        if constexpr (kList)
            return useg_decode(a.L, raw);
        else
            return useg_dense(a, s < nseg ? s : 0, segs_x, ny_b);
    };
    // one body: a second inlined copy of the operators would overflow the instruction cache.
    // Counts run two segments ahead of the sweep and the loads one segment ahead; the copies
    // (cur = nxt, c1 = cfar) happen a whole finish() after their loads were issued.
    USeg cur, nxt;
    UPre pre;
    {
        const USegId id0 = locate(warp, kList ? useg_raw(a, warp, nseg, n1) : 0u);
        useg_issue<kTwoInline, kWrap>(a, id0, lane, useg_count(a, id0, true, lane), nxt);
    }
    USegId idfar = locate(warp + nwarps, kList ? useg_raw(a, warp + nwarps, nseg, n1) : 0u);
    int cfar = useg_count(a, idfar, warp + nwarps < nseg, lane);
    unsigned rawfar = kList ? useg_raw(a, warp + 2 * nwarps, nseg, n1) : 0u;
    for (long long s = warp; s < nseg; s += nwarps) {
        cur = nxt;
        useg_pre<kVsnap, kTwoInline>(a, cur, pre);
        const int c1 = cfar;
        const USegId id1 = idfar;
        idfar = locate(s + 2 * nwarps, rawfar);
        cfar = useg_count(a, idfar, s + 2 * nwarps < nseg, lane);
        if constexpr (kList) rawfar = useg_raw(a, s + 3 * nwarps, nseg, n1);
        if (s + nwarps < nseg) useg_issue<kTwoInline, kWrap>(a, id1, lane, c1, nxt);
        useg_finish<kFused, kVsnap, kTwoInline>(a, cur, pre);
    }
}

// K12, TMA-fed (LBG_K12_TMA=1; unforced, non-fused, direct snapshot index, unwrapped blocks):
// the register-pipelined kernel above keeps the next segment's 19 populations and cell fields
// in registers (166 registers, 3 CTAs of 4 warps per SM) and still waits for them in most of
// its stall samples. Here each warp owns kTStages shared-memory stages, filled by 1-D bulk
// copies (one per pulled q-row, issued by lanes 0..18 in parallel, plus the btot / b0 / pidx0
// windows of a covered segment by lanes 19..21) completing on the stage's mbarrier — nothing in
// flight occupies registers or the LSU. The row windows are the sectors the lanes' pulls touch
// and no more: [i0, i0 + 32) for c_x = 0, [i0 - 2, i0 + 32) for c_x = +1 (pull from x - 1),
// [i0, i0 + 34) for c_x = -1 (16-byte aligned starts). The lanes store their count bytes
// (loaded one segment before the copies are issued) into the stage. The consumer rebuilds the
// USeg from the stage and runs the same useg_pre / useg_finish as the register-pipelined
// kernel, so the results are bitwise the same.
struct TStage {
    double f[kQ][34];
    double bt[34];
    double b0[34];
    int pe[36];
    int cnt[32];
    int mx, pad[3];
};
static_assert(sizeof(TStage) % 16 == 0, "TMA stage must keep 16-byte alignment");
constexpr int kTWarps = 4;   // warps per CTA
constexpr int kTStages = 2;  // stages per warp

__host__ __device__ constexpr size_t tma_smem_bytes() {
    return sizeof(TStage) * kTStages * kTWarps + sizeof(unsigned long long) * kTStages * kTWarps;
}

// the row window of population q: first element (relative to i0) and bytes
__device__ __forceinline__ int trow_first(int q) { return cx(q) == 1 ? -2 : 0; }
__device__ __forceinline__ unsigned trow_bytes(int q) { return cx(q) == 0 ? 256u : 272u; }
// index of lane l's pulled value (x = i0 + l - c_x) in its row window
__device__ __forceinline__ int trow_at(int q, int l) { return l - cx(q) - trow_first(q); }

// the whole warp: the copies of segment `id` (warp max count mx) into `st`; lane q < 19 copies
// row q
__device__ __forceinline__ void tseg_issue(const SweepArgs& a, const USegId& id, int mx, TStage& st,
                                           unsigned long long* bar, int lane) {
    const Layout& L = a.L;
    // lane q: the offset of its row window from the segment's cell index, and its size
    // (compile-time per q: a select chain, no local-memory table)
    long long roff = 0;
    unsigned rbytes = 0;
#pragma unroll
    for (int q = 0; q < kQ; ++q)
        if (lane == q) {
            roff = (long long)q * L.plane + trow_first(q) - cy(q) * (long long)L.px -
                   cz(q) * (long long)L.px * L.py;
            rbytes = trow_bytes(q);
        }
    const long long c = L.frac(id.i0, id.j, id.k);
    const long long c2 = c & ~1LL, c4 = c & ~3LL;
    const unsigned bb = (unsigned)(((c + 32 - c2) + 1) & ~1LL) * 8u;  // 256 or 272
    const unsigned pb = (unsigned)(((c + 32 - c4) + 3) & ~3LL) * 4u;  // 128 .. 144
    if (lane == 0) {
        unsigned tx = 9u * 256u + 10u * 272u;
        if (mx >= 1) tx += 2u * bb + pb;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the consumer's reads of st
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
                     : "memory");
    }
    __syncwarp();
    if (lane < kQ) {
        tma_bulk(&st.f[0][0] + 34 * lane, a.src + (L.idx(id.i0, id.j, id.k) + roff), rbytes, bar);
    } else if (mx >= 1) {
        if (lane == kQ) tma_bulk(st.bt, a.btot + c2, bb, bar);
        if (lane == kQ + 1) tma_bulk(st.b0, a.b0 + c2, bb, bar);
        if (lane == kQ + 2) tma_bulk(st.pe, a.pidx0 + c4, pb, bar);
    }
}

template <bool kVsnap>
__global__ void __launch_bounds__(32 * kTWarps, 4) coupled_tma_kernel(const SweepArgs a) {
    extern __shared__ __align__(128) unsigned char tsm[];
    const Layout& L = a.L;
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const long long warp = (long long)blockIdx.x * kTWarps + wl;
    const long long nwarps = (long long)gridDim.x * kTWarps;
    const int segs_x = (a.hi[0] - a.i0 + 31) >> 5;
    const int ny_b = a.hi[1] - a.lo[1];
    const long long nseg = (long long)segs_x * ny_b * (a.hi[2] - a.lo[2]);
    TStage* st = reinterpret_cast<TStage*>(tsm) + kTStages * wl;
    unsigned long long* bar =
        reinterpret_cast<unsigned long long*>(tsm + sizeof(TStage) * kTStages * kTWarps) + kTStages * wl;
    if (warp >= nseg) return;  // warp-uniform
    if (lane == 0) {
        for (int t = 0; t < kTStages; ++t)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[t])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    // issue segment s into stage t: counts into the stage (this lane's), the copies
    auto issue = [&](long long s, int cnt, int t) {
        const USegId id = useg_dense(a, s, segs_x, ny_b);
        const int mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
        st[t].cnt[lane] = cnt;
        if (lane == 0) st[t].mx = mx;
        tseg_issue(a, id, mx, st[t], &bar[t], lane);
    };
    // prologue: the first kTStages segments in flight, the counts of the next one loaded
#pragma unroll
    for (int t = 0; t < kTStages; ++t) {
        const long long s = warp + t * nwarps;
        if (s < nseg) issue(s, useg_count(a, useg_dense(a, s, segs_x, ny_b), true, lane), t);
    }
    long long sfar = warp + kTStages * nwarps;
    int cfar = useg_count(a, useg_dense(a, sfar < nseg ? sfar : 0, segs_x, ny_b), sfar < nseg, lane);
    unsigned phase = 0;  // bit t: parity of stage t
    int t = 0;
    for (long long s = warp; s < nseg; s += nwarps) {
        {
            unsigned done = 0;
            const unsigned par = (phase >> t) & 1u;
            do {
                asm volatile(
                    "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                    " selp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done)
                    : "r"(smem_u32(&bar[t])), "r"(par)
                    : "memory");
            } while (!done);
            phase ^= 1u << t;
        }
        __syncwarp();  // the lanes' count stores of this stage are visible
        // rebuild the segment from the stage
        USeg u;
        {
            const TStage& S = st[t];
            const USegId id = useg_dense(a, s, segs_x, ny_b);
            u.i = id.i0 + lane;
            u.j = id.j;
            u.k = id.k;
            const bool inx = u.i < L.nx;
            u.fc = LBG_IDX(L.frac(inx ? u.i : L.nx - 1, u.j, u.k), a.cells, a.err);
            u.act = inx && u.i >= a.lo[0] && u.i < a.hi[0];
            u.cnt = S.cnt[lane];
            u.mx = S.mx;
            const long long c0 = L.frac(id.i0, id.j, id.k);
            if (u.mx >= 1) {
                u.bt = S.bt[lane + (int)(c0 & 1)];
                u.b0 = S.b0[lane + (int)(c0 & 1)];
                u.pe = S.pe[lane + (int)(c0 & 3)];
            }
            if (u.mx >= 2) {  // two-entry segment (rare): entry 1 from global
                u.b1 = a.b1[u.fc];
                u.id1 = a.id1[u.fc];
            }
            u.base = LBG_IDX(L.idx(u.i, u.j, u.k), L.plane, a.err);
#pragma unroll
            for (int q = 0; q < kQ; ++q) u.f[q] = S.f[q][trow_at(q, lane)];
        }
        UPre pre;
        useg_pre<kVsnap, true>(a, u, pre);
        // the next count set (one segment ahead of its copies)
        const int c1 = cfar;
        const long long s1 = sfar;
        sfar += nwarps;
        cfar = useg_count(a, useg_dense(a, sfar < nseg ? sfar : 0, segs_x, ny_b), sfar < nseg, lane);
        __syncwarp();  // every lane has read stage t
        if (s1 < nseg) issue(s1, c1, t);
        useg_finish<false, kVsnap, true>(a, u, pre);
        t = (t + 1 == kTStages) ? 0 : t + 1;
    }
}

// Thin boxes of a coupled block (the boundary shell), split like K1/K2 by the operator a cell
// needs rather than by segment: kTwo = false sweeps every shell cell with count <= 1 (the
// ~94-register one-entry path), kTwo = true only the two-entry cells (general operator), so
// the heavy operator's registers never limit the bulk of the shell.
template <bool kForced, bool kFused, bool kTwo, bool kVsnap>
__global__ void __launch_bounds__(128) sweep_flat_coupled_kernel(const SweepArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    double m[2][3] = {{0, 0, 0}, {0, 0, 0}};
    double cc[3] = {0, 0, 0};
    int p0 = -1, p1 = -1;
    if (t < a.bstart[a.nbox]) {
        int i, j, k;
        flat_cell(a, t, i, j, k);
        const long long fc = a.L.frac(i, j, k);
        const int cnt = a.count[fc];
        if (kTwo ? cnt > 1 : cnt <= 1)
            ok = coupled_lane<kForced, kFused, kTwo, kVsnap>(a, i, j, k, fc, cnt, m, p0, p1, cc);
    }
    count_bad(a.err, !ok);
    if constexpr (kFused) {
        fused_accumulate(a, p0, m[0], cc);
        fused_accumulate(a, p1, m[1], cc);
    }
}

// lbm.cpp:6-17 — unfused pull stream.
__global__ void stream_kernel(const double* __restrict__ src, double* __restrict__ dst, Layout L,
                              int lo0, int lo1, int lo2, int hi0, int hi1) {
    const int i = lo0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int j = lo1 + blockIdx.y;
    const int k = lo2 + blockIdx.z;
    if (i >= hi0 || j >= hi1) return;
    const long long base = L.idx(i, j, k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) dst[q * L.plane + base] = src[q * L.plane + base - L.shift(q)];
}

#ifdef LBG_CHECKED
// every cell of the sweep's boxes written exactly once, no other cell written; counts reset
__global__ void __launch_bounds__(256) verify_writes_kernel(SweepArgs a) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= a.cells) return;
    const int i = (int)(c % a.L.nx), j = (int)((c / a.L.nx) % a.L.ny), k = (int)(c / ((long long)a.L.nx * a.L.ny));
    const int want = in_boxes(a, i, j, k) ? 1 : 0;
    if (a.wc[c] != want) atomicAdd(&a.err->race, 1ull);
    a.wc[c] = 0;
}
#endif

static lbg_status verify_writes(lbg_block b, const SweepArgs& a) {
#ifdef LBG_CHECKED
    verify_writes_kernel<<<(unsigned)((a.cells + 255) / 256), 256, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
#else
    (void)b;
    (void)a;
#endif
    return LBG_OK;
}

static lbg_status ensure_wcount(lbg_block b) {
#ifdef LBG_CHECKED
    if (!b->wcount) {
        const size_t n = (size_t)b->L.nx * b->L.ny * b->L.nz;
        LBG_CUDA(cudaMalloc(&b->wcount, sizeof(int) * n));
        LBG_CUDA(cudaMemset(b->wcount, 0, sizeof(int) * n));
    }
#else
    (void)b;
#endif
    return LBG_OK;
}

static bool valid_box(const Layout& L, const lbg_box& r) {
    const int d[3] = {L.nx, L.ny, L.nz};
    for (int a = 0; a < 3; ++a)
        if (r.lo[a] < 0 || r.hi[a] > d[a]) return false;
    return true;
}

static bool empty_box(const lbg_box& r) {
    return r.hi[0] <= r.lo[0] || r.hi[1] <= r.lo[1] || r.hi[2] <= r.lo[2];
}

// LBG_DIRECT_INDEX=0: the inline solid velocity always goes through id0 -> id table (A/B)
static bool lbg_direct_index_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("LBG_DIRECT_INDEX");
        return !(e && e[0] == '0');
    }();
    return v;
}

// the fused force mode needs its per-particle accumulators for the current snapshot list
static lbg_status check_fused(lbg_block b) {
    if (b->coupling && b->force_mode == LBG_FORCE_FUSED && b->n_snaps > 0 &&
        (!b->facc || !b->fused_used || b->facc_cap < b->n_snaps))
        return set_error(LBG_INVALID, "fused force mode without accumulators for the snapshot list");
    return LBG_OK;
}

static SweepArgs make_args(lbg_block b, const lbg_fluid* fl) {
    SweepArgs a{};
    a.src = b->src();
    a.dst = b->dst();
    a.L = b->L;
    a.inv_tau = 1.0 / fl->tau;  // kDt / params.tau (lbm.cpp:30)
    a.F = {fl->f_ext[0], fl->f_ext[1], fl->f_ext[2]};
    a.err = b->err_d;
    a.wc = b->wcount;
    a.cells = (long long)b->L.nx * b->L.ny * b->L.nz;
    for (int c = 0; c < 3; ++c) a.wrap[c] = b->wrap[c];
    if (b->coupling) {
        a.count = b->count;
        a.b0 = b->b0;
        a.b1 = b->b1;
        a.btot = b->btot;
        a.v0 = b->v0;
        a.v1 = b->v1;
        a.m0 = b->m0;
        a.m1 = b->m1;
        a.seg_list = b->seg_list;
        a.seg_n = b->seg_n;
        a.seg_cap = b->seg_cap;
        a.id0 = b->id0;
        a.id1 = b->id1;
        a.snaps = b->snaps_d;
        a.n_snaps = b->n_snaps;
        a.sidx = snap_index(b);
        a.pidx0 = (b->v_snap && b->p_direct && lbg_direct_index_enabled()) ? b->pidx0 : nullptr;
        for (int c = 0; c < 3; ++c) a.blk_lo[c] = b->lo[c];
        a.facc = b->facc;
        a.fused_used = b->fused_used;
    }
    return a;
}

static lbg_status add_boxes(SweepArgs& a, const Layout& L, const lbg_box* boxes, int n) {
    a.nbox = 0;
    a.bstart[0] = 0;
    for (int t = 0; t < n; ++t) {
        if (empty_box(boxes[t])) continue;
        if (!valid_box(L, boxes[t])) return set_error(LBG_INVALID, "sweep range outside the block");
        long long vol = 1;
        for (int c = 0; c < 3; ++c) {
            a.blo[a.nbox][c] = boxes[t].lo[c];
            a.bext[a.nbox][c] = boxes[t].hi[c] - boxes[t].lo[c];
            vol *= a.bext[a.nbox][c];
        }
        a.bstart[a.nbox + 1] = a.bstart[a.nbox] + vol;
        ++a.nbox;
    }
    return LBG_OK;
}

template <bool kForced, bool kSkip>
static void launch_box(const SweepArgs& a, cudaStream_t s) {
    constexpr int BX = 128, BY = 2;
    dim3 block(BX, BY, 1);
    dim3 grid((a.hi[0] - a.i0 + BX - 1) / BX, (a.hi[1] - a.lo[1] + BY - 1) / BY, a.hi[2] - a.lo[2]);
    sweep_box_kernel<kForced, kSkip><<<grid, block, 0, s>>>(a);
}

template <bool kForced>
static void launch_pair(SweepArgs a, cudaStream_t s) {
    constexpr int BY = 8;
    a.i0 = (a.lo[0] / 64) * 64;
    dim3 block(32, BY, 1);
    dim3 grid((a.hi[0] - a.i0 + 63) / 64, (a.hi[1] - a.lo[1] + BY - 1) / BY, a.hi[2] - a.lo[2]);
    sweep_pair_kernel<kForced><<<grid, block, 0, s>>>(a);
}

// K1 variant for plain blocks: the one-cell-per-lane kernel (default) or, with
// LBG_SWEEP_PAIR=1, the 128-bit pair kernel. Measured on B200 at 512^3 (profiles/
// r01_sweep_ab.txt): 6.28 ms vs 6.40 ms per sweep — both at the HBM roofline (99.2 % / 97.5 %
// of the measured copy bandwidth); the pair kernel's 2x bytes per lane come with half the
// resident warps (128 vs 70 registers), so the 64-bit coalesced kernel stays the default.
static bool pair_sweep() {
    static const bool v = [] {
        const char* e = std::getenv("LBG_SWEEP_PAIR");
        return e && e[0] == '1';
    }();
    return v;
}

template <bool kForced, bool kSkip>
static void launch_flat(const SweepArgs& a, cudaStream_t s) {
    const long long n = a.bstart[a.nbox];
    const int T = 256;
    sweep_flat_kernel<kForced, kSkip><<<(unsigned)((n + T - 1) / T), T, 0, s>>>(a);
}

// calls fn(std::bool_constant<x>, std::bool_constant<y>, std::bool_constant<z>): runtime
// flags to kernel template arguments
template <class Fn>
static void with_flags(bool x, bool y, bool z, Fn&& fn) {
    auto zf = [&](auto X, auto Y) { z ? fn(X, Y, std::true_type{}) : fn(X, Y, std::false_type{}); };
    auto yf = [&](auto X) { y ? zf(X, std::true_type{}) : zf(X, std::false_type{}); };
    x ? yf(std::true_type{}) : yf(std::false_type{});
}

// unforced one-entry K2 variant, LBG_K2_MODE: 0 plain segment loop, 1 register-pipelined,
// 2 TMA-fed (profiles/r01_ab_k2.txt)
static int k2_mode() {
    static const int v = [] {
        const char* e = std::getenv("LBG_K2_MODE");
        return e ? std::atoi(e) : 1;
    }();
    return v;
}

static int k2_tma_per_sm() {
    static const int v = [] {
        const char* e = std::getenv("LBG_K2_TMA_SM");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    return v;
}

static int k2_pipe_per_sm() {
    static const int v = [] {
        const char* e = std::getenv("LBG_K2_PIPE_SM");
        return e ? std::max(1, std::atoi(e)) : 3;
    }();
    return v;
}

// K2 on stream `st`, `per_sm` persistent CTAs of 128 per SM for the one-entry segments
static void launch_psm_segments(lbg_block b, const SweepArgs& a, bool forced, cudaStream_t st, int per_sm) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
    const bool fused = b->force_mode == LBG_FORCE_FUSED;
    const unsigned g1 = (unsigned)(sms * per_sm), g2 = (unsigned)(sms * 4);
    with_flags(forced, fused, b->v_snap, [&](auto F, auto U, auto V) {
        // segments with one-entry cells only (the bulk): lean pair-scheduled operator
        if (!decltype(F)::value && k2_mode() == 2) {
            constexpr size_t smem = (sizeof(SegStage) + 8) * 2 * kTmaWarps;
            auto kern = psm_seg_tma_kernel<decltype(U)::value, decltype(V)::value>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<(unsigned)(sms * k2_tma_per_sm()), 32 * kTmaWarps, smem, st>>>(a);
        } else if (!decltype(F)::value && k2_mode() == 1)
            psm_seg_pipe_kernel<decltype(U)::value, decltype(V)::value>
                <<<(unsigned)(sms * k2_pipe_per_sm()), 128, 0, st>>>(a);
        else
            psm_seg_kernel<decltype(F)::value, decltype(U)::value, false, decltype(V)::value><<<g1, 128, 0, st>>>(a);
        count_launch();
        // segments holding a two-entry cell (particle contacts): general operator
        psm_seg_kernel<decltype(F)::value, decltype(U)::value, true, decltype(V)::value><<<g2, 128, 0, st>>>(a);
    });
}

// K12 (coupled_unified_kernel) settings: LBG_K12=0 restores the K1 || K2 split, LBG_K12_SM =
// CTAs per SM (4, 5 or 6: also the register cap; 5 measured best)
static int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
static bool k12_on() {
    static const bool v = env_int("LBG_K12", 1) != 0;
    return v;
}

template <bool kForced, bool kSkip>
static void launch_box(const SweepArgs& a, cudaStream_t s);

// Coupled sweep kernel choice (LBG_K12): 0 round 1's K1 || K2 split; 2 the unified kernel; 3 the
// covered-list split (K1 over the segments without a covered cell, K12 over the mapping's
// covered-segment list); 1 (default) picks 2 or 3 by the block's covered fraction of the last
// mapping: above LBG_K12_SPLIT_BELOW (default 0.35) the unified kernel (config 3's dense bed,
// 62 % covered segments: 1.03 ms vs 1.13 split), below it the split (config 5's dilute bed,
// ~12 %: 6.7 ms vs 8.0 unified; profiles/r02_ab_k12.txt)
static int k12_mode() {
    static const int v = env_int("LBG_K12", 1);
    return v;
}

// the covered fraction of the block's segments, from the counts the last mapping posted (-1
// while they are not on the host yet)
static double covered_fraction(lbg_block b) {
    if (!b->segn_pending || !b->segn_h || !b->ev_segn) return -1.0;
    if (cudaEventQuery(b->ev_segn) != cudaSuccess) {
        cudaGetLastError();  // cudaErrorNotReady is not an error
        return -1.0;
    }
    const double total = (double)((b->L.nx + 31) / 32) * b->L.ny * b->L.nz;
    return total > 0 ? (b->segn_h[0] + b->segn_h[1]) / total : 0.0;
}

static void launch_unified(lbg_block b, const SweepArgs& a, bool forced, cudaStream_t st) {
    static const int per_sm = std::min(6, std::max(4, env_int("LBG_K12_SM", 5)));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
    const bool fused = b->force_mode == LBG_FORCE_FUSED;
    const long long nseg = (long long)((a.hi[0] - a.i0 + 31) / 32) * (a.hi[1] - a.lo[1]) * (a.hi[2] - a.lo[2]);
    with_flags(forced, fused, b->v_snap, [&](auto F, auto U, auto V) {
        constexpr bool kF = decltype(F)::value, kU = decltype(U)::value, kV = decltype(V)::value;
        auto go = [&](auto kern, int ctas) {
            const long long want = (nseg + 3) / 4;  // CTAs of 4 warps, one segment each
            const unsigned grid = (unsigned)std::max(1LL, std::min<long long>(want, (long long)sms * ctas));
            kern<<<grid, 128, 0, st>>>(a);
        };
        static const int pipe = env_int("LBG_K12_PIPE", 1);
        static const int two_inline = env_int("LBG_K12_TWO", 1);
        static const int nowrap = env_int("LBG_K12_NOWRAP", 1);  // 0: the generic pull (A/B)
        const bool wrapped = a.wrap[0] || a.wrap[1] || a.wrap[2] || !nowrap;
        static const int tma = env_int("LBG_K12_TMA", 0);
        if (!kF && !kU && pipe && a.pidx0 && two_inline && tma && !wrapped) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(coupled_tma_kernel<kV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tma_smem_bytes());
                attr = true;
            }
            const long long want = (nseg + kTWarps - 1) / kTWarps;
            const unsigned grid = (unsigned)std::max(1LL, std::min<long long>(want, (long long)sms * 4));
            coupled_tma_kernel<kV><<<grid, 32 * kTWarps, tma_smem_bytes(), st>>>(a);
            return;
        }
        if (!kF && pipe && a.pidx0 && two_inline) {
            if (wrapped)
                go(coupled_unified_pipe_kernel<kU, kV, true, true>, LBG_K12_MINB);
            else
                go(coupled_unified_pipe_kernel<kU, kV, true, false>, LBG_K12_MINB);
            return;  // every segment swept by the one kernel
        }
        if (!kF && pipe && a.pidx0)
            go(coupled_unified_pipe_kernel<kU, kV, false, true>, LBG_K12_MINB);
        else if (kF || per_sm == 4)
            go(coupled_unified_kernel<kF, kU, kV, 4>, 4);
        else if (per_sm == 6)
            go(coupled_unified_kernel<kF, kU, kV, 6>, 6);
        else
            go(coupled_unified_kernel<kF, kU, kV, 5>, 5);
        count_launch();
        // segments holding a two-entry cell (particle contacts): pair-scheduled two-entry operator
        psm_seg_kernel<kF, kU, true, kV><<<(unsigned)(sms * 4), 128, 0, st>>>(a);
    });
}

// K12 over the covered-segment list only (unforced, direct snapshot index): one- and
// two-entry segments, the pipelined operator loop
static void launch_covered_list(lbg_block b, const SweepArgs& a, cudaStream_t st) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
    const bool fused = b->force_mode == LBG_FORCE_FUSED;
    const bool wrapped = a.wrap[0] || a.wrap[1] || a.wrap[2];
    const unsigned grid = (unsigned)(sms * LBG_K12_MINB);
    with_flags(fused, b->v_snap, wrapped, [&](auto U, auto V, auto W) {
        constexpr bool kU = decltype(U)::value, kV = decltype(V)::value, kW = decltype(W)::value;
        coupled_unified_pipe_kernel<kU, kV, true, kW, true><<<grid, 128, 0, st>>>(a);
    });
}

// LBG_K2_CONCURRENT=0 runs K2 after K1 on the compute stream (A/B measurement)
static bool k2_concurrent() {
    static const bool v = [] {
        const char* e = std::getenv("LBG_K2_CONCURRENT");
        return !(e && e[0] == '0');
    }();
    return v;
}

// K1 over the z-planes [z0, z1) (whole x/y extent) of a plain block from `src` into `dst` on
// stream `st`: the streamed host job's sweeps (lbg_job.cu), which alternate two buffers per
// step instead of lbg_swap
lbg_status sweep_planes(lbg_block b, const lbg_fluid* fl, const double* src, double* dst, int z0, int z1,
                        cudaStream_t st) {
    if (z1 <= z0) return LBG_OK;
    if (lbg_status s = ensure_wcount(b)) return s;
    SweepArgs a = make_args(b, fl);
    a.src = src;
    a.dst = dst;
    a.lo[0] = a.lo[1] = 0;
    a.hi[0] = b->L.nx;
    a.hi[1] = b->L.ny;
    a.lo[2] = z0;
    a.hi[2] = z1;
    a.i0 = 0;
    const lbg_box box = {{0, 0, z0}, {b->L.nx, b->L.ny, z1}};
    if (lbg_status s = add_boxes(a, b->L, &box, 1)) return s;
    const bool fo = fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
    fo ? launch_box<true, false>(a, st) : launch_box<false, false>(a, st);
    LBG_LAUNCH_CHECK();
    return verify_writes(b, a);
}

}  // namespace lbg

using namespace lbg;

static lbg_status check_fluid(const lbg_fluid* fl) {
    if (!fl) return set_error(LBG_INVALID, "null fluid params");
    if (!(fl->tau > 0.5))  // FluidParams::validate (lbm.hpp:28-32)
        return set_error(LBG_CONFIG_ERROR, "fluid relaxation time tau must be > 0.5 (got " +
                                               std::to_string(fl->tau) + ")");
    return LBG_OK;
}

static bool forced(const lbg_fluid* fl) {
    return fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
}

extern "C" {

lbg_status lbg_sweep(lbg_block b, const lbg_fluid* fl, const lbg_box* range) {
    if (!b || !range) return set_error(LBG_INVALID, "null argument");
    if (lbg_status s = check_fluid(fl)) return s;
    if (empty_box(*range)) return LBG_OK;  // run_kernel skips empty ranges (sim.cpp:222)
    if (!valid_box(b->L, *range)) return set_error(LBG_INVALID, "sweep range outside the block");
    LBG_CUDA(cudaSetDevice(b->device));
    if (b->aa) {  // AA in-place streaming: whole block, every axis wrapped
        if (range->lo[0] != 0 || range->lo[1] != 0 || range->lo[2] != 0 || range->hi[0] != b->L.nx ||
            range->hi[1] != b->L.ny || range->hi[2] != b->L.nz)
            return set_error(LBG_INVALID, "AA streaming sweeps the whole block");
        if (!(b->wrap[0] && b->wrap[1] && b->wrap[2]))
            return set_error(LBG_INVALID, "AA streaming needs the in-kernel periodic wrap on every axis");
        if (b->aa_pending) return set_error(LBG_INVALID, "AA streaming: lbg_swap between sweeps");
        Span span(b, LBG_CAT_PSM);
        return aa_sweep(b, fl);
    }
    if (b->coupling && b->cov_dirty)
        if (lbg_status s = rebuild_covered(b)) return s;
    if (lbg_status s = check_fused(b)) return s;
    if (lbg_status s = ensure_wcount(b)) return s;
    SweepArgs a = make_args(b, fl);
    for (int c = 0; c < 3; ++c) {
        a.lo[c] = range->lo[c];
        a.hi[c] = range->hi[c];
    }
    a.i0 = (range->lo[0] / 32) * 32;
    if (lbg_status s = add_boxes(a, b->L, range, 1)) return s;
    Span span(b, LBG_CAT_PSM);
    const bool fo = forced(fl);
    // a coupled block mapped from an empty particle list has count 0 everywhere: the PSM sweep
    // is collide_cell in every cell (psm.cpp:236-240), so it is the plain K1 sweep exactly
    const bool no_cover = b->coupling && b->v_snap && b->map_ids_valid && b->map_ids.empty() && !b->cov_dirty;
    if (no_cover) {
        fo ? launch_box<true, false>(a, b->stream) : launch_box<false, false>(a, b->stream);
        LBG_LAUNCH_CHECK();
        return verify_writes(b, a);
    }
    if (b->coupling) {
        if (k12_on()) {
            static const double split_below = [] {
                const char* e = std::getenv("LBG_K12_SPLIT_BELOW");
                return e ? std::atof(e) : 0.35;
            }();
            const int mode = k12_mode();
            const double cf = mode == 1 ? covered_fraction(b) : -1.0;
            const bool list_ok = !fo && a.pidx0;
            if (list_ok && (mode == 3 || (mode == 1 && cf >= 0.0 && cf < split_below))) {
                // K1 over the fluid segments, then K12 over the covered-segment list
                launch_box<false, true>(a, b->stream);
                LBG_LAUNCH_CHECK();
                launch_covered_list(b, a, b->stream);
                LBG_LAUNCH_CHECK();
                return verify_writes(b, a);
            }
            launch_unified(b, a, fo, b->stream);
            LBG_LAUNCH_CHECK();
            return verify_writes(b, a);
        }
        if (k2_concurrent()) {
            // K1 and K2 touch disjoint cells (K1 skips K2's segments): K2 runs on the aux stream
            // beside K1, with fewer persistent CTAs so K1's blocks find room on every SM
            LBG_CUDA(cudaEventRecord(b->ev_fork, b->stream));
            LBG_CUDA(cudaStreamWaitEvent(b->aux, b->ev_fork, 0));
            launch_psm_segments(b, a, fo, b->aux, 4);
            LBG_LAUNCH_CHECK();
            fo ? launch_box<true, true>(a, b->stream) : launch_box<false, true>(a, b->stream);
            LBG_LAUNCH_CHECK();
            LBG_CUDA(cudaEventRecord(b->ev_join, b->aux));
            LBG_CUDA(cudaStreamWaitEvent(b->stream, b->ev_join, 0));
            return verify_writes(b, a);
        }
        fo ? launch_box<true, true>(a, b->stream) : launch_box<false, true>(a, b->stream);
        LBG_LAUNCH_CHECK();
        launch_psm_segments(b, a, fo, b->stream, 8);
    } else if (pair_sweep()) {
        fo ? launch_pair<true>(a, b->stream) : launch_pair<false>(a, b->stream);
    } else {
        fo ? launch_box<true, false>(a, b->stream) : launch_box<false, false>(a, b->stream);
    }
    LBG_LAUNCH_CHECK();
    return verify_writes(b, a);
}

lbg_status lbg_sweep_boxes(lbg_block b, const lbg_fluid* fl, const lbg_box* boxes, int n) {
    if (lbg_status s_ = aa_refuse(b, "lbg_sweep_boxes")) return s_;
    if (!b || (!boxes && n > 0)) return set_error(LBG_INVALID, "null argument");
    if (lbg_status s = check_fluid(fl)) return s;
    if (n > 8) return set_error(LBG_INVALID, "at most 8 boxes per launch");
    LBG_CUDA(cudaSetDevice(b->device));
    if (b->coupling && b->cov_dirty)
        if (lbg_status s = rebuild_covered(b)) return s;
    if (lbg_status s = check_fused(b)) return s;
    if (lbg_status s = ensure_wcount(b)) return s;
    SweepArgs a = make_args(b, fl);
    if (lbg_status s = add_boxes(a, b->L, boxes, n)) return s;
    if (a.nbox == 0) return LBG_OK;
    Span span(b, LBG_CAT_PSM);
    const bool fo = forced(fl);
    if (b->coupling) {
        const long long n_cells = a.bstart[a.nbox];
        const unsigned grid = (unsigned)((n_cells + 127) / 128);
        const bool fu = b->force_mode == LBG_FORCE_FUSED;
        with_flags(fo, fu, b->v_snap, [&](auto F, auto U, auto V) {
            constexpr bool kF = decltype(F)::value, kU = decltype(U)::value, kV = decltype(V)::value;
            sweep_flat_coupled_kernel<kF, kU, false, kV><<<grid, 128, 0, b->stream>>>(a);
            count_launch();
            sweep_flat_coupled_kernel<kF, kU, true, kV><<<grid, 128, 0, b->stream>>>(a);
        });
    } else {
        fo ? launch_flat<true, false>(a, b->stream) : launch_flat<false, false>(a, b->stream);
    }
    LBG_LAUNCH_CHECK();
    return verify_writes(b, a);
}

lbg_status lbg_stream(lbg_block b, const lbg_box* r) {
    if (lbg_status s_ = aa_refuse(b, "lbg_stream")) return s_;
    if (!b || !r) return set_error(LBG_INVALID, "null argument");
    if (empty_box(*r)) return LBG_OK;
    if (!valid_box(b->L, *r)) return set_error(LBG_INVALID, "stream range outside the block");
    LBG_CUDA(cudaSetDevice(b->device));
    dim3 grid((r->hi[0] - r->lo[0] + 127) / 128, r->hi[1] - r->lo[1], r->hi[2] - r->lo[2]);
    stream_kernel<<<grid, 128, 0, b->stream>>>(b->src(), b->dst(), b->L, r->lo[0], r->lo[1],
                                                r->lo[2], r->hi[0], r->hi[1]);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

}  // extern "C"
