// SPDX-License-Identifier: Apache-2.0
//
// K1/K2 — fused pull-stream + SRT (+PSM) collide sweep over a CellBox.
//   reference: collide_stream_impl (lbm.cpp:21-49), psm_collide_stream_impl (psm.cpp:218-262)
//
// Roofline: HBM-bound. Algorithmic bytes per lattice update (LUP): 19 f64 pulled + 19 f64
// stored = 304 B for the plain sweep; the coupled sweep adds the 1-byte count per cell and,
// per covered cell, 8 B btot + per entry (8 B b + 24 B v read, 24 B m written).
//
// Launch shapes:
//   box  — one CellBox, 3-D grid; thread x maps to global i with the chunk origin aligned to
//          32 cells, so every warp's loads/stores of a q-plane are two 128-B lines
//          (the pulled x-neighbour costs one extra sector per warp, served by L1/L2).
//   flat — up to 8 boxes in one launch (the 6 boundary_shell boxes of field.cpp:55-72),
//          flattened cell index; used for thin boxes where a 3-D grid would idle lanes.
// Unstable cells (lbm.hpp:106) are counted with a warp ballot into the block's error
// counter; lbg_sync() raises NumericError like the reference does after the sweep.
#include "lbg_cell.cuh"
#include "lbg_internal.cuh"

namespace lbg {

struct SweepArgs {
    const double* __restrict__ src;
    double* __restrict__ dst;
    Layout L;
    double inv_tau;
    Force F;
    DeviceErrors* err;
    // coupling (interior lexicographic)
    const uint8_t* __restrict__ count;
    const double* __restrict__ b0;
    const double* __restrict__ b1;
    const double* __restrict__ btot;
    const double* __restrict__ v0;
    const double* __restrict__ v1;
    double* __restrict__ m0;
    double* __restrict__ m1;
    // box launch
    int lo[3], hi[3];
    int i0;  // aligned chunk origin
    // flat launch
    int nbox;
    int blo[8][3];
    int bext[8][3];
    long long bstart[9];
};

template <bool kForced, bool kCoupled>
__device__ __forceinline__ bool process_cell(const SweepArgs& a, int i, int j, int k) {
    const Layout& L = a.L;
    const long long base = L.idx(i, j, k);
    double f[kQ];
#pragma unroll
    for (int q = 0; q < kQ; ++q) f[q] = a.src[q * L.plane + base - L.shift(q)];

    bool ok;
    if constexpr (kCoupled) {
        const long long fc = L.frac(i, j, k);
        const int cnt = a.count[fc];
        if (cnt == 0) {
            ok = srt_cell<kForced>(f, a.inv_tau, a.F);
        } else {
            const double be[2] = {a.b0[fc], cnt > 1 ? a.b1[fc] : 0.0};
            double ue[2][3];
            for (int c = 0; c < 3; ++c) {
                ue[0][c] = a.v0[3 * fc + c];
                ue[1][c] = cnt > 1 ? a.v1[3 * fc + c] : 0.0;
            }
            double m[2][3];
            ok = psm_cell(f, a.inv_tau, a.F, cnt, a.btot[fc], be, ue, m);
            for (int c = 0; c < 3; ++c) a.m0[3 * fc + c] = m[0][c];
            if (cnt > 1)
                for (int c = 0; c < 3; ++c) a.m1[3 * fc + c] = m[1][c];
        }
    } else {
        ok = srt_cell<kForced>(f, a.inv_tau, a.F);
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) a.dst[q * L.plane + base] = f[q];
    return ok;
}

__device__ __forceinline__ void count_bad(DeviceErrors* err, bool bad) {
    const unsigned m = __ballot_sync(0xffffffffu, bad);
    if (m && (threadIdx.x & 31) == 0) atomicAdd(&err->unstable, (unsigned long long)__popc(m));
}

template <bool kForced, bool kCoupled>
__global__ void __launch_bounds__(256) sweep_box_kernel(const SweepArgs a) {
    const int i = a.i0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int j = a.lo[1] + blockIdx.y * blockDim.y + threadIdx.y;
    const int k = a.lo[2] + blockIdx.z;
    const bool active = i >= a.lo[0] && i < a.hi[0] && j < a.hi[1];
    bool ok = true;
    if (active) ok = process_cell<kForced, kCoupled>(a, i, j, k);
    count_bad(a.err, !ok);
}

template <bool kForced, bool kCoupled>
__global__ void __launch_bounds__(256) sweep_flat_kernel(const SweepArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (t < a.bstart[a.nbox]) {
        int b = 0;
        while (t >= a.bstart[b + 1]) ++b;
        const long long r = t - a.bstart[b];
        const int ex = a.bext[b][0], ey = a.bext[b][1];
        const int i = a.blo[b][0] + (int)(r % ex);
        const int j = a.blo[b][1] + (int)((r / ex) % ey);
        const int k = a.blo[b][2] + (int)(r / ((long long)ex * ey));
        ok = process_cell<kForced, kCoupled>(a, i, j, k);
    }
    count_bad(a.err, !ok);
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

static bool valid_box(const Layout& L, const lbg_box& r) {
    const int d[3] = {L.nx, L.ny, L.nz};
    for (int a = 0; a < 3; ++a)
        if (r.lo[a] < 0 || r.hi[a] > d[a]) return false;
    return true;
}

static bool empty_box(const lbg_box& r) {
    return r.hi[0] <= r.lo[0] || r.hi[1] <= r.lo[1] || r.hi[2] <= r.lo[2];
}

static SweepArgs make_args(lbg_block b, const lbg_fluid* fl) {
    SweepArgs a{};
    a.src = b->src();
    a.dst = b->dst();
    a.L = b->L;
    a.inv_tau = 1.0 / fl->tau;  // kDt / params.tau (lbm.cpp:30)
    a.F = {fl->f_ext[0], fl->f_ext[1], fl->f_ext[2]};
    a.err = b->err_d;
    if (b->coupling) {
        a.count = b->count;
        a.b0 = b->b0;
        a.b1 = b->b1;
        a.btot = b->btot;
        a.v0 = b->v0;
        a.v1 = b->v1;
        a.m0 = b->m0;
        a.m1 = b->m1;
    }
    return a;
}

template <bool kForced, bool kCoupled>
static void launch_box(const SweepArgs& a, cudaStream_t s) {
    constexpr int BX = 128, BY = 2;
    dim3 block(BX, BY, 1);
    dim3 grid((a.hi[0] - a.i0 + BX - 1) / BX, (a.hi[1] - a.lo[1] + BY - 1) / BY, a.hi[2] - a.lo[2]);
    sweep_box_kernel<kForced, kCoupled><<<grid, block, 0, s>>>(a);
}

template <bool kForced, bool kCoupled>
static void launch_flat(const SweepArgs& a, cudaStream_t s) {
    const long long n = a.bstart[a.nbox];
    const int T = 256;
    sweep_flat_kernel<kForced, kCoupled><<<(unsigned)((n + T - 1) / T), T, 0, s>>>(a);
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

extern "C" {

lbg_status lbg_sweep(lbg_block b, const lbg_fluid* fl, const lbg_box* range) {
    if (!b || !range) return set_error(LBG_INVALID, "null argument");
    if (lbg_status s = check_fluid(fl)) return s;
    if (empty_box(*range)) return LBG_OK;  // run_kernel skips empty ranges (sim.cpp:222)
    if (!valid_box(b->L, *range)) return set_error(LBG_INVALID, "sweep range outside the block");
    LBG_CUDA(cudaSetDevice(b->device));
    SweepArgs a = make_args(b, fl);
    for (int c = 0; c < 3; ++c) {
        a.lo[c] = range->lo[c];
        a.hi[c] = range->hi[c];
    }
    a.i0 = (range->lo[0] / 32) * 32;
    const bool forced = fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
    Span span(b, LBG_CAT_PSM);
    if (b->coupling) {
        forced ? launch_box<true, true>(a, b->stream) : launch_box<false, true>(a, b->stream);
    } else {
        forced ? launch_box<true, false>(a, b->stream) : launch_box<false, false>(a, b->stream);
    }
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_sweep_boxes(lbg_block b, const lbg_fluid* fl, const lbg_box* boxes, int n) {
    if (!b || (!boxes && n > 0)) return set_error(LBG_INVALID, "null argument");
    if (lbg_status s = check_fluid(fl)) return s;
    if (n > 8) return set_error(LBG_INVALID, "at most 8 boxes per launch");
    LBG_CUDA(cudaSetDevice(b->device));
    SweepArgs a = make_args(b, fl);
    a.nbox = 0;
    a.bstart[0] = 0;
    for (int t = 0; t < n; ++t) {
        if (empty_box(boxes[t])) continue;
        if (!valid_box(b->L, boxes[t])) return set_error(LBG_INVALID, "sweep range outside the block");
        long long vol = 1;
        for (int c = 0; c < 3; ++c) {
            a.blo[a.nbox][c] = boxes[t].lo[c];
            a.bext[a.nbox][c] = boxes[t].hi[c] - boxes[t].lo[c];
            vol *= a.bext[a.nbox][c];
        }
        a.bstart[a.nbox + 1] = a.bstart[a.nbox] + vol;
        ++a.nbox;
    }
    if (a.nbox == 0) return LBG_OK;
    const bool forced = fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
    Span span(b, LBG_CAT_PSM);
    if (b->coupling) {
        forced ? launch_flat<true, true>(a, b->stream) : launch_flat<false, true>(a, b->stream);
    } else {
        forced ? launch_flat<true, false>(a, b->stream) : launch_flat<false, false>(a, b->stream);
    }
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_stream(lbg_block b, const lbg_box* r) {
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
