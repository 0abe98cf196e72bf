// SPDX-License-Identifier: Apache-2.0
//
// AA-pattern in-place streaming (lbg_set_streaming(LBG_STREAM_AA)) — one PDF buffer instead
// of the reference's two (PdfField::src/dst + swap, field.hpp:36-78): half the HBM per block.
//
// States of the single buffer (slot q of cell x = plane q at x):
//   S0 (after an even number of AA steps): slot q of x holds the post-collision f*_q(x) — the
//      double-buffer src exactly, so switching to AA from a double-buffered state is free.
//   S1 (after an odd number): slot q̄ of x holds the population arriving at x in direction q
//      (f*_q(x - c_q), streamed, pre-collision).
// Odd step (S0 -> S1): cell y pulls f_q = slot q at y - c_q (the double-buffer pull), collides
// (srt_cell, unchanged) and stores f**_q(y) into slot q̄ at y + c_q — the slot y itself read for
// q̄, so every thread overwrites exactly its own 19 reads and no two threads touch one slot.
// Even step (S1 -> S0): cell x reads f_q = slot q̄ at x, collides, stores slot q at x.
// The collision of every cell sees the same 19 values as the pull sweep, so the populations are
// bitwise those of the double-buffered path. Periodic wrap in-kernel on every axis (the slots a
// boundary cell touches across a face are the wrapped interior ones; no ghost layer is read or
// written): single-block periodic plain-fluid blocks (configs 1-2). Roofline: 304 B per LUP
// either way; the even step's accesses are all unshifted.
#include <cstdlib>

#include "lbg_cell.cuh"
#include "lbg_internal.cuh"

namespace lbg {

struct AAArgs {
    // the one buffer, passed twice: with one pointer the compiler keeps the 19 load addresses
    // live for the stores (124 registers); as two it recomputes them (70, like K1)
    const double* buf_r;
    double* buf_w;
    Layout L;
    double inv_tau;
    Force F;
    DeviceErrors* err;
};

// offset of slot q of cell (i, j, k) + c_q * sgn, every axis wrapped
__device__ __forceinline__ long long aa_off(const Layout& L, int i, int j, int k, int q, int sgn) {
    int x = i + sgn * cx(q), y = j + sgn * cy(q), z = k + sgn * cz(q);
    x = x < 0 ? L.nx - 1 : (x >= L.nx ? 0 : x);
    y = y < 0 ? L.ny - 1 : (y >= L.ny ? 0 : y);
    z = z < 0 ? L.nz - 1 : (z >= L.nz ? 0 : z);
    return q * L.plane + L.idx(x, y, z);
}

template <bool kForced, bool kOdd>
__global__ void __launch_bounds__(256) sweep_aa_kernel(const AAArgs a) {
    const Layout& L = a.L;
    // read and write views of the one buffer: every value a thread stores depends on all 19 it
    // loaded (the density), so no store can precede a load of the same slot, and no two threads
    // touch one slot — the views never alias in any order the compiler can produce
    const double* __restrict__ rd = a.buf_r;
    double* __restrict__ wr = a.buf_w;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int k = blockIdx.z;
    bool ok = true;
    if (i < L.nx && j < L.ny) {
        double f[kQ];
        const long long base = L.idx(i, j, k);
        // odd step: the wrapped neighbour coordinates once per cell; the 9 (dy, dz) rows D3Q19
        // reaches serve both the pulls (x - c_q) and the stores (x + c_q)
        int xs[3] = {i == 0 ? L.nx - 1 : i - 1, i, i == L.nx - 1 ? 0 : i + 1};
        int ys[3] = {j == 0 ? L.ny - 1 : j - 1, j, j == L.ny - 1 ? 0 : j + 1};
        int zs[3] = {k == 0 ? L.nz - 1 : k - 1, k, k == L.nz - 1 ? 0 : k + 1};
        auto at = [&](int q, int sgn) {  // slot q of the cell at (i, j, k) + sgn * c_q
            return (long long)q * L.plane + L.row(ys[1 + sgn * cy(q)], zs[1 + sgn * cz(q)]) + xs[1 + sgn * cx(q)];
        };
        if (kOdd) {
#pragma unroll
            for (int q = 0; q < kQ; ++q) f[q] = rd[at(q, -1)];
        } else {
#pragma unroll
            for (int q = 0; q < kQ; ++q) f[q] = rd[opposite(q) * L.plane + base];
        }
        ok = srt_cell<kForced>(f, a.inv_tau, a.F);
        if (kOdd) {
            // the store addresses are the load addresses of the opposite populations: make the
            // coordinates opaque here so they are recomputed rather than held in 38 registers
            asm volatile("" : "+r"(xs[0]), "+r"(xs[1]), "+r"(xs[2]), "+r"(ys[0]), "+r"(ys[1]), "+r"(ys[2]),
                         "+r"(zs[0]), "+r"(zs[1]), "+r"(zs[2]));
#pragma unroll
            for (int q = 0; q < kQ; ++q) wr[at(opposite(q), -1)] = f[q];
        } else {
#pragma unroll
            for (int q = 0; q < kQ; ++q) wr[q * L.plane + base] = f[q];
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, !ok);
    if (m && (threadIdx.x & 31) == 0) atomicAdd(&a.err->unstable, (unsigned long long)__popc(m));
}

// S1 -> S0 without a collision: slot q of x in `out` = slot q̄ of x + c_q in `in` (where the odd
// step stored x's post-collision f_q); `in` and `out` distinct
__global__ void __launch_bounds__(256) aa_unstream_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                          Layout L) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    if (i >= L.nx) return;
    const long long base = L.idx(i, j, k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) out[q * L.plane + base] = in[aa_off(L, i, j, k, opposite(q), -1)];
}

lbg_status aa_sweep(lbg_block b, const lbg_fluid* fl) {
    AAArgs a{};
    a.buf_r = b->buf[b->cur];
    a.buf_w = b->buf[b->cur];
    a.L = b->L;
    a.inv_tau = 1.0 / fl->tau;  // lbm.cpp:30
    a.F = {fl->f_ext[0], fl->f_ext[1], fl->f_ext[2]};
    a.err = b->err_d;
    const bool forced = fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
    const bool odd = b->aa_phase == 0;  // S0 -> S1
    // CTAs of 256 threads along x (LBG_AA_BX = 128/64/32 for A/B: 256 measured best, the odd
    // step's x-shifted stores then split fewer lines between CTAs; profiles/r02_ab_k12.txt)
    static const int bx = [] {
        const char* e = std::getenv("LBG_AA_BX");
        const int v = e ? std::atoi(e) : 256;
        return (v == 32 || v == 64 || v == 128) ? v : 256;
    }();
    const int by = 256 / bx;
    dim3 block(bx, by, 1);
    dim3 grid((b->L.nx + bx - 1) / bx, (b->L.ny + by - 1) / by, b->L.nz);
    if (forced)
        odd ? sweep_aa_kernel<true, true><<<grid, block, 0, b->stream>>>(a)
            : sweep_aa_kernel<true, false><<<grid, block, 0, b->stream>>>(a);
    else
        odd ? sweep_aa_kernel<false, true><<<grid, block, 0, b->stream>>>(a)
            : sweep_aa_kernel<false, false><<<grid, block, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
    b->aa_pending = true;  // lbg_swap completes the step (phase flip)
    return LBG_OK;
}

// the S0 image of an S1 buffer into `out` (a full PDF buffer)
lbg_status aa_unstream(lbg_block b, double* out) {
    dim3 grid((b->L.nx + 127) / 128, b->L.ny, b->L.nz);
    aa_unstream_kernel<<<grid, 128, 0, b->stream>>>(b->buf[b->cur], out, b->L);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

}  // namespace lbg

using namespace lbg;

extern "C" {

lbg_status lbg_set_streaming(lbg_block b, int mode) {
    if (!b) return set_error(LBG_INVALID, "null block");
    if (mode != LBG_STREAM_AB && mode != LBG_STREAM_AA) return set_error(LBG_INVALID, "bad streaming mode");
    LBG_CUDA(cudaSetDevice(b->device));
    if ((mode == LBG_STREAM_AA) == b->aa) return LBG_OK;
    const size_t pdf_bytes = sizeof(double) * (kQ * (size_t)b->L.plane + 128);
    if (mode == LBG_STREAM_AA) {
        if (b->coupling || b->comm || b->p2p || b->push)
            return set_error(LBG_INVALID, "AA streaming is the single-block plain-fluid path (no coupling, no halo)");
        // the double-buffer src is state S0: keep it, release the other buffer
        LBG_CUDA(cudaStreamSynchronize(b->stream));
        LBG_CUDA(cudaFree(b->buf[b->cur ^ 1]));
        b->buf[b->cur ^ 1] = nullptr;
        b->device_bytes -= (long long)pdf_bytes;
        b->aa = true;
        b->aa_phase = 0;
        b->aa_pending = false;
        return LBG_OK;
    }
    // back to two buffers: the S0 image goes into the new one when the state is S1
    double* nb = nullptr;
    LBG_CUDA(cudaMalloc(&nb, pdf_bytes));
    LBG_CUDA(cudaMemsetAsync(nb, 0, pdf_bytes, b->stream));
    b->device_bytes += (long long)pdf_bytes;
    if (b->aa_phase == 1) {
        if (lbg_status s = aa_unstream(b, nb)) return s;
        LBG_CUDA(cudaStreamSynchronize(b->stream));
        std::swap(b->buf[b->cur], nb);
        b->buf[b->cur ^ 1] = nb;  // the old S1 buffer becomes dst
    } else {
        b->buf[b->cur ^ 1] = nb;
    }
    b->aa = false;
    b->aa_phase = 0;
    return LBG_OK;
}

}  // extern "C"
