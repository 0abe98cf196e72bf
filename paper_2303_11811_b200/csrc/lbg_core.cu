// SPDX-License-Identifier: Apache-2.0
//
// liblbg core: block lifecycle (BlockState/PdfField, sim.cpp:15-25, field.cpp:6-35),
// host<->device transfers in the reference layout, the end-of-phase sync with the
// reference's error semantics, observers and per-category CUDA-event timing
// (perf::Category, perf.hpp:17-26).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>

#include "lbg_internal.cuh"

namespace lbg {

namespace {
thread_local std::string g_last_error;
std::atomic<long long> g_launches{0};
}  // namespace

lbg_status set_error(lbg_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

lbg_status cuda_check(cudaError_t e, const char* what) {
    return set_error(LBG_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static cudaEvent_t take_event(lbg_block b) {
    if (!b->event_pool.empty()) {
        cudaEvent_t e = b->event_pool.back();
        b->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

Span::Span(lbg_block b_, int cat_) : b(b_), cat(cat_) {
    if (b->timing) {
        a = take_event(b);
        cudaEventRecord(a, b->stream);
    }
}

Span::~Span() {
    if (a) {
        cudaEvent_t e = take_event(b);
        cudaEventRecord(e, b->stream);
        b->spans.push_back({cat, a, e});
    }
}

// lbm.hpp:38-45 — host twin of equilibrium() with the reference's operation order
// (this TU is compiled with -ffp-contract=off for the host side).
static void equilibrium_host(double rho, const double u[3], double feq[kQ]) {
    const double u_sq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int q = 0; q < kQ; ++q) {
        const double c0 = cx(q), c1 = cy(q), c2 = cz(q);
        const double cu = c0 * u[0] + c1 * u[1] + c2 * u[2];
        feq[q] = wq(q) * (rho + 1.0 * (cu * 3.0 + 0.5 * cu * cu * 9.0 - 0.5 * u_sq * 3.0));
    }
}

struct Feq {
    double v[kQ];
};

__global__ void fill_interior_kernel(double* __restrict__ buf, Layout L, Feq f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    if (i >= L.nx) return;
    const long long c = L.idx(i, j, k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) buf[q * L.plane + c] = f.v[q];
}

// validation.cpp:46-63 shear-wave initial state, evaluated per cell on the device
// (synthetic benchmark input; device sin/cos may differ from glibc in the last ulp).
__global__ void shear_wave_kernel(double* __restrict__ buf, Layout L, int lo0, int lo1, int lo2, int D0,
                                  int D1, int D2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int k = blockIdx.z;
    if (i >= L.nx) return;
    const double pi = 3.14159265358979323846;
    const double gx = lo0 + i + 0.5, gy = lo1 + j + 0.5, gz = lo2 + k + 0.5;
    const double u0 = 0.02 * sin(2.0 * pi * gy / D1);
    const double u1 = 0.015 * cos(2.0 * pi * gz / D2);
    const double u2 = 0.01 * sin(2.0 * pi * gx / D0);
    const double u_sq = (u0 * u0 + u1 * u1) + u2 * u2;
    const long long c = L.idx(i, j, k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double cu = ((double)cx(q) * u0 + (double)cy(q) * u1) + (double)cz(q) * u2;
        buf[q * L.plane + c] = wq(q) * (1.0 + 1.0 * ((cu * 3.0 + ((0.5 * cu) * cu) * 9.0) - (0.5 * u_sq) * 3.0));
    }
}

__global__ void fill_ghosts_kernel(double* __restrict__ buf, Layout L, double v) {
    // all cells of the (nx+2)(ny+2)(nz+2) box that are not interior
    const int ii = blockIdx.x * blockDim.x + threadIdx.x;  // 0..nx+1
    const int jj = blockIdx.y;
    const int kk = blockIdx.z;
    if (ii >= L.nx + 2) return;
    const int i = ii - 1, j = jj - 1, k = kk - 1;
    const bool interior = i >= 0 && i < L.nx && j >= 0 && j < L.ny && k >= 0 && k < L.nz;
    if (interior) return;
    const long long c = L.idx(i, j, k);
#pragma unroll
    for (int q = 0; q < kQ; ++q) buf[q * L.plane + c] = v;
}

// Row-wise Neumaier partial sums of the src interior (lbm.cpp:69-93), combined on the
// host in lexicographic row order.
__device__ __forceinline__ void nm_add(double& sum, double& comp, double v) {
    const double t = sum + v;
    if (fabs(sum) >= fabs(v))
        comp += (sum - t) + v;
    else
        comp += (v - t) + sum;
    sum = t;
}

__global__ void row_moments_kernel(const double* __restrict__ src, Layout L, double* __restrict__ rows) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;  // j + k*ny
    if (row >= L.ny * L.nz) return;
    const int j = row % L.ny, k = row / L.ny;
    double s[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0};
    const long long base = L.row(j, k);
    for (int i = 0; i < L.nx; ++i) {
        double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const double f = src[q * L.plane + base + i];
            rho += f;
            mx += f * (double)cx(q);
            my += f * (double)cy(q);
            mz += f * (double)cz(q);
        }
        nm_add(s[0], c[0], rho);
        nm_add(s[1], c[1], mx);
        nm_add(s[2], c[2], my);
        nm_add(s[3], c[3], mz);
    }
    for (int a = 0; a < 4; ++a) {
        rows[(size_t)row * 8 + 2 * a] = s[a];
        rows[(size_t)row * 8 + 2 * a + 1] = c[a];
    }
}

// ---- per-step observers (output.cpp:22-61 sample_scalars; lbm.cpp:69-93), on the device.
// Each thread walks a fixed strided set of cells with Neumaier accumulators, the CTA combines
// the (sum, comp) pairs in a fixed tree, and the host adds the CTA partials in order:
// deterministic for a given grid (not bitwise equal to the reference's serial order).
constexpr int kObsThreads = 256;
constexpr int kObsVals = 5;  // mass, px, py, pz, fluid KE

__device__ __forceinline__ void two_sum_add(double& s, double& c, double s2, double c2) {
    const double t = s + s2;
    const double bp = t - s;
    const double err = (s - (t - bp)) + (s2 - bp);
    s = t;
    c = (c + c2) + err;
}

__global__ void __launch_bounds__(kObsThreads) observe_kernel(const double* __restrict__ src, Layout L,
                                                               double fx, double fy, double fz,
                                                               double* __restrict__ part) {
    double s[kObsVals] = {0, 0, 0, 0, 0}, c[kObsVals] = {0, 0, 0, 0, 0};
    double max_u2 = 0.0;
    const long long cells = (long long)L.nx * L.ny * L.nz;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < cells;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % L.nx), j = (int)((t / L.nx) % L.ny), k = (int)(t / ((long long)L.nx * L.ny));
        const long long base = L.idx(i, j, k);
        double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const double f = src[q * L.plane + base];
            rho += f;
            mx += f * (double)cx(q);
            my += f * (double)cy(q);
            mz += f * (double)cz(q);
        }
        // lbm.hpp:55-63: observable velocity carries the half-force shift
        const double ux = mx / 1.0 + (1.0 / (2.0 * 1.0)) * fx;
        const double uy = my / 1.0 + (1.0 / (2.0 * 1.0)) * fy;
        const double uz = mz / 1.0 + (1.0 / (2.0 * 1.0)) * fz;
        const double u2 = (ux * ux + uy * uy) + uz * uz;
        const double v[kObsVals] = {rho, mx, my, mz, 0.5 * rho * u2};
#pragma unroll
        for (int a = 0; a < kObsVals; ++a) nm_add(s[a], c[a], v[a]);
        max_u2 = fmax(max_u2, u2);
    }
    __shared__ double sh[kObsThreads / 32][2 * kObsVals + 1];
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int a = 0; a < kObsVals; ++a) {
            const double s2 = __shfl_down_sync(0xffffffffu, s[a], o);
            const double c2 = __shfl_down_sync(0xffffffffu, c[a], o);
            two_sum_add(s[a], c[a], s2, c2);
        }
        max_u2 = fmax(max_u2, __shfl_down_sync(0xffffffffu, max_u2, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        for (int a = 0; a < kObsVals; ++a) {
            sh[w][2 * a] = s[a];
            sh[w][2 * a + 1] = c[a];
        }
        sh[w][2 * kObsVals] = max_u2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double* out = part + (size_t)blockIdx.x * (2 * kObsVals + 1);
        for (int a = 0; a < kObsVals; ++a) {
            double ss = sh[0][2 * a], cc = sh[0][2 * a + 1];
            for (int v = 1; v < kObsThreads / 32; ++v) two_sum_add(ss, cc, sh[v][2 * a], sh[v][2 * a + 1]);
            out[2 * a] = ss;
            out[2 * a + 1] = cc;
        }
        double m = sh[0][2 * kObsVals];
        for (int v = 1; v < kObsThreads / 32; ++v) m = fmax(m, sh[v][2 * kObsVals]);
        out[2 * kObsVals] = m;
    }
}

// ---- per-cell moments for observers and grid dumps (lbm.hpp:55-63 macroscopic before the
// f_ext shift, lbm.cpp:61-93): rho = 0 + f_0 + ... + f_18 and m = 0 + f_q c_q in q order,
// i.e. the reference's own sums (the c_q = 0 terms add a signed zero to a partial sum that
// starts at +0, which never changes it). One thread per cell of a z-chunk, AoS output in the
// reference's lexicographic cell order; btot appended when the block is coupled.
__global__ void moments_kernel(const double* __restrict__ src, Layout L, int k0, int nk,
                               const double* __restrict__ btot, int with_frac, double* __restrict__ out) {
    const long long slice = (long long)L.nx * L.ny;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= slice * nk) return;
    const int i = (int)(t % L.nx), j = (int)((t / L.nx) % L.ny), k = k0 + (int)(t / slice);
    const long long base = L.idx(i, j, k);
    double rho = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double f = src[q * L.plane + base];
        rho += f;
        if (cx(q) == 1) mx += f; else if (cx(q) == -1) mx -= f;
        if (cy(q) == 1) my += f; else if (cy(q) == -1) my -= f;
        if (cz(q) == 1) mz += f; else if (cz(q) == -1) mz -= f;
    }
    const int stride = with_frac ? 5 : 4;
    double* o = out + t * stride;
    o[0] = rho;
    o[1] = mx;
    o[2] = my;
    o[3] = mz;
    if (with_frac) o[4] = btot ? btot[k * slice + (long long)j * L.nx + i] : 0.0;
}

}  // namespace lbg

using namespace lbg;

extern "C" {

lbg_status lbg_observe(lbg_block b, const double f_ext[3], double out[6]) {
    if (lbg_status s_ = aa_refuse(b, "lbg_observe", true)) return s_;
    if (!b || !out) return set_error(LBG_INVALID, "null argument");
    LBG_CUDA(cudaSetDevice(b->device));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, b->device);
    const int blocks = sms * 4;
    const size_t per = 2 * kObsVals + 1;
    if (!b->obs_d || !b->obs_h) {
        size_t cap = 0;
        if (lbg_status s = grow_device(b->obs_d, cap, (long long)(per * blocks), (long long)(per * blocks),
                                       "cudaMalloc(observers)"))
            return s;
        if (!b->obs_h) LBG_CUDA(cudaMallocHost(&b->obs_h, sizeof(double) * per * blocks));
    }
    const double fx = f_ext ? f_ext[0] : 0.0, fy = f_ext ? f_ext[1] : 0.0, fz = f_ext ? f_ext[2] : 0.0;
    {
        Span span(b, LBG_CAT_OTHER);
        observe_kernel<<<blocks, kObsThreads, 0, b->stream>>>(b->src(), b->L, fx, fy, fz, b->obs_d);
        LBG_LAUNCH_CHECK();
        LBG_CUDA(cudaMemcpyAsync(b->obs_h, b->obs_d, sizeof(double) * per * blocks, cudaMemcpyDeviceToHost,
                                 b->stream));
    }
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    double s[kObsVals] = {0, 0, 0, 0, 0}, c[kObsVals] = {0, 0, 0, 0, 0}, mx = 0.0;
    for (int k = 0; k < blocks; ++k) {
        const double* p = b->obs_h + per * k;
        for (int a = 0; a < kObsVals; ++a) {
            const double t = s[a] + p[2 * a];
            if (std::fabs(s[a]) >= std::fabs(p[2 * a]))
                c[a] += (s[a] - t) + p[2 * a];
            else
                c[a] += (p[2 * a] - t) + s[a];
            s[a] = t;
            c[a] += p[2 * a + 1];
        }
        mx = std::max(mx, p[2 * kObsVals]);
    }
    for (int a = 0; a < kObsVals; ++a) out[a] = s[a] + c[a];
    out[5] = std::sqrt(mx);
    return LBG_OK;
}

lbg_status lbg_moments(lbg_block b, int with_frac, double* out) {
    if (lbg_status s_ = aa_refuse(b, "lbg_moments", true)) return s_;
    if (!b || !out) return set_error(LBG_INVALID, "null argument");
    LBG_CUDA(cudaSetDevice(b->device));
    const Layout& L = b->L;
    const int stride = with_frac ? 5 : 4;
    const long long slice = (long long)L.nx * L.ny;
    // z-chunks of at most ~64 MB staged on the device, copied out on the compute stream
    const long long kz = std::max(1LL, std::min<long long>(L.nz, (8LL << 20) / (slice * stride)));
    const size_t bytes = sizeof(double) * (size_t)(kz * slice * stride);
    if (lbg_status s = grow_device(b->mom_d, b->mom_cap, (long long)(bytes / sizeof(double)),
                                   (long long)(bytes / sizeof(double)), "cudaMalloc(moments)"))
        return s;
    Span span(b, LBG_CAT_OTHER);
    for (long long k0 = 0; k0 < L.nz; k0 += kz) {
        const int nk = (int)std::min<long long>(kz, L.nz - k0);
        const long long n = slice * nk;
        moments_kernel<<<(unsigned)((n + 255) / 256), 256, 0, b->stream>>>(
            b->src(), L, (int)k0, nk, with_frac ? b->btot : nullptr, with_frac, b->mom_d);
        LBG_LAUNCH_CHECK();
        LBG_CUDA(cudaMemcpyAsync(out + k0 * slice * stride, b->mom_d, sizeof(double) * n * stride,
                                 cudaMemcpyDeviceToHost, b->stream));
    }
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

const char* lbg_last_error(void) { return g_last_error.c_str(); }
const char* lbg_version(void) {
#ifdef LBG_CHECKED
    return "lbg 0.2 (sm_100a, checked)";
#else
    return "lbg 0.2 (sm_100a)";
#endif
}

int lbg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

lbg_status lbg_host_alloc(size_t bytes, void** out) {
    LBG_CUDA(cudaMallocHost(out, bytes));
    return LBG_OK;
}

lbg_status lbg_host_free(void* p) {
    LBG_CUDA(cudaFreeHost(p));
    return LBG_OK;
}

long long lbg_launch_count(void) { return g_launches.load(); }

lbg_status lbg_block_create(int device, const int box_lo[3], const int dims[3], int coupling,
                            lbg_block* out) {
    *out = nullptr;
    for (int a = 0; a < 3; ++a)
        if (dims[a] < 1) return set_error(LBG_CONFIG_ERROR, "block dimensions must be positive");
    LBG_CUDA(cudaSetDevice(device));
    auto* b = new lbg_block_s;
    b->device = device;
    for (int a = 0; a < 3; ++a) b->lo[a] = box_lo[a];
    b->coupling = coupling != 0;
    Layout& L = b->L;
    L.nx = dims[0];
    L.ny = dims[1];
    L.nz = dims[2];
    L.px = ((kXOff + L.nx + 1) + 15) / 16 * 16;
    L.py = L.ny + 2;
    L.pz = L.nz + 2;
    L.plane = (long long)L.px * L.py * L.pz;

    auto fail = [&](cudaError_t e, const char* what) {
        lbg_block_destroy(b);
        return cuda_check(e, what);
    };
    // + slack: the TMA-fed K2 copies 40-double row windows that may run past the last row
    const size_t pdf_bytes = sizeof(double) * (kQ * (size_t)L.plane + 128);
    cudaError_t e;
    for (int s = 0; s < 2; ++s) {
        if ((e = cudaMalloc(&b->buf[s], pdf_bytes)) != cudaSuccess) return fail(e, "cudaMalloc(pdf)");
        if ((e = cudaMemset(b->buf[s], 0, pdf_bytes)) != cudaSuccess) return fail(e, "cudaMemset(pdf)");
        b->device_bytes += pdf_bytes;
    }
    if (b->coupling) {
        // + 64 cells of slack: the TMA-fed K2 copies 34/36/48-element field windows per segment
        const size_t n = (size_t)L.nx * L.ny * L.nz + 64;
        struct A {
            void** p;
            size_t bytes;
        } allocs[] = {{(void**)&b->count, n},
                      {(void**)&b->id0, n * 4},
                      {(void**)&b->id1, n * 4},
                      {(void**)&b->pidx0, n * 4},
                      {(void**)&b->b0, n * 8},
                      {(void**)&b->b1, n * 8},
                      {(void**)&b->btot, n * 8},
                      {(void**)&b->v0, n * 24},
                      {(void**)&b->v1, n * 24},
                      {(void**)&b->m0, n * 24},
                      {(void**)&b->m1, n * 24}};
        for (auto& a : allocs) {
            if ((e = cudaMalloc(a.p, a.bytes)) != cudaSuccess) return fail(e, "cudaMalloc(coupling)");
            if ((e = cudaMemset(*a.p, 0, a.bytes)) != cudaSuccess) return fail(e, "cudaMemset(coupling)");
            b->device_bytes += a.bytes;
        }
        // FractionField::resize fills id0/id1 with -1 (field.cpp:37-46)
        cudaMemset(b->id0, 0xff, n * 4);
        cudaMemset(b->id1, 0xff, n * 4);
        b->seg_cap = (long long)((L.nx + 31) / 32) * L.ny * L.nz;
        if ((e = cudaMalloc(&b->seg_list, sizeof(unsigned) * b->seg_cap)) != cudaSuccess) return fail(e, "cudaMalloc(seg)");
        if ((e = cudaMalloc(&b->seg_n, 2 * sizeof(int))) != cudaSuccess) return fail(e, "cudaMalloc(seg_n)");
        cudaMemset(b->seg_n, 0, 2 * sizeof(int));
        b->cov_dirty = false;  // all-zero count: empty list
        b->device_bytes += sizeof(unsigned) * n;
    }
    if ((e = cudaMalloc(&b->err_d, sizeof(DeviceErrors))) != cudaSuccess) return fail(e, "cudaMalloc(err)");
    cudaMemset(b->err_d, 0, sizeof(DeviceErrors));
    if ((e = cudaMallocHost(&b->err_h, sizeof(DeviceErrors))) != cudaSuccess) return fail(e, "cudaMallocHost(err)");
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if ((e = cudaStreamCreateWithPriority(&b->stream, cudaStreamNonBlocking, lo_prio)) != cudaSuccess)
        return fail(e, "cudaStreamCreate");
    if ((e = cudaStreamCreateWithPriority(&b->side, cudaStreamNonBlocking, hi_prio)) != cudaSuccess)
        return fail(e, "cudaStreamCreate(side)");
    if ((e = cudaStreamCreateWithPriority(&b->aux, cudaStreamNonBlocking, lo_prio)) != cudaSuccess)
        return fail(e, "cudaStreamCreate(aux)");
    if ((e = cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "cudaEventCreate(fork/join)");
    if ((e = cudaEventCreateWithFlags(&b->ev_side, cudaEventDisableTiming)) != cudaSuccess)
        return fail(e, "cudaEventCreate");
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e, "block create");
    *out = b;
    return LBG_OK;
}

lbg_status lbg_comm_destroy(lbg_block b);  // lbg_halo.cu
lbg_status lbg_p2p_destroy(lbg_block b);   // lbg_p2p.cu
lbg_status lbg_halo_push_destroy(lbg_block b);  // lbg_push.cu

lbg_status lbg_block_destroy(lbg_block b) {
    if (!b) return LBG_OK;
    cudaSetDevice(b->device);
    if (b->stream) cudaStreamSynchronize(b->stream);
    if (b->side) cudaStreamSynchronize(b->side);
    if (b->aux) cudaStreamSynchronize(b->aux);
    if (b->comm) lbg_comm_destroy(b);
    if (b->p2p) lbg_p2p_destroy(b);
    if (b->push) lbg_halo_push_destroy(b);
    lbg::free_shadow(b);
    void* dev[] = {b->buf[0], b->buf[1], b->count, b->id0, b->id1, b->b0, b->b1, b->btot,
                   b->v0, b->v1, b->m0, b->m1, b->snaps_d, b->bin_count, b->bin_start,
                   b->bin_items, b->red_rows, b->red_used, b->err_d, b->facc, b->fused_used,
                   b->obs_d, b->mom_d, b->seg_list, b->seg_n, b->snap_tab, b->red_box, b->pidx0, b->wcount, b->bin_rec};
    for (void* p : dev)
        if (p) cudaFree(p);
    void* host[] = {b->snaps_h, b->err_h, b->red_rows_h, b->red_used_h, b->obs_h, b->segn_h};
    for (void* p : host)
        if (p) cudaFreeHost(p);
    for (auto& s : b->spans) {
        cudaEventDestroy(s.a);
        cudaEventDestroy(s.b);
    }
    for (auto e : b->event_pool) cudaEventDestroy(e);
    if (b->ev_side) cudaEventDestroy(b->ev_side);
    if (b->ev_fork) cudaEventDestroy(b->ev_fork);
    if (b->ev_join) cudaEventDestroy(b->ev_join);
    if (b->ev_stage) cudaEventDestroy(b->ev_stage);
    if (b->ev_fetched) cudaEventDestroy(b->ev_fetched);
    if (b->ev_red) cudaEventDestroy(b->ev_red);
    if (b->ev_segn) cudaEventDestroy(b->ev_segn);
    for (int s = 0; s < 2; ++s) {
        if (b->xfer[s]) cudaFree(b->xfer[s]);
        if (b->ev_copy[s]) cudaEventDestroy(b->ev_copy[s]);
        if (b->ev_done[s]) cudaEventDestroy(b->ev_done[s]);
    }
    lbg::free_job(b);
    for (double* p : b->stage)
        if (p) cudaFree(p);
    if (b->recv_buf) cudaFree(b->recv_buf);
    for (double* p : b->recv_multi)
        if (p) cudaFree(p);
    if (b->stream) cudaStreamDestroy(b->stream);
    if (b->side) cudaStreamDestroy(b->side);
    if (b->aux) cudaStreamDestroy(b->aux);
    delete b;
    return LBG_OK;
}

lbg_status lbg_block_info(lbg_block b, int dims[3], int box_lo[3], int* coupling,
                          long long* device_bytes) {
    if (!b) return set_error(LBG_INVALID, "null block");
    if (dims) {
        dims[0] = b->L.nx;
        dims[1] = b->L.ny;
        dims[2] = b->L.nz;
    }
    if (box_lo)
        for (int a = 0; a < 3; ++a) box_lo[a] = b->lo[a];
    if (coupling) *coupling = b->coupling;
    if (device_bytes) *device_bytes = b->device_bytes;
    return LBG_OK;
}

void* lbg_block_stream(lbg_block b) { return b ? (void*)b->stream : nullptr; }

// packed reference rows (stride nx+2) <-> pitched device rows (stride px, offset kXOff-1)
__global__ void repitch_kernel(double* __restrict__ dev, const double* __restrict__ packed_in,
                               double* __restrict__ packed_out, long long row0, long long rows, int w,
                               int px) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * w) return;
    const long long r = t / w;
    const int c = (int)(t % w);
    double* d = dev + (row0 + r) * px + (kXOff - 1) + c;
    if (packed_in)
        *d = packed_in[t];
    else
        packed_out[t] = *d;
}

// Large transfers from/to PINNED host memory: linear chunk copies on the side stream (full
// PCIe rate) double-buffered against the re-pitch kernel on the compute stream, instead of one
// row-by-row 2-D copy.
static lbg_status copy_pdf_pinned(lbg_block b, double* dev, const double* host_in, double* host_out) {
    const Layout& L = b->L;
    const int w = L.nx + 2;
    const long long rows = (long long)kQ * L.py * L.pz;
    const long long chunk_rows = std::max<long long>(1, (256ll << 20) / (8ll * w));
    const size_t chunk_bytes = sizeof(double) * (size_t)chunk_rows * w;
    if (!b->xfer[0] || !b->xfer[1]) {
        for (int s = 0; s < 2; ++s) {
            size_t cap = 0;
            if (lbg_status st = grow_device(b->xfer[s], cap, (long long)(chunk_bytes / sizeof(double)),
                                            (long long)(chunk_bytes / sizeof(double)), "cudaMalloc(transfer staging)"))
                return st;
            if (!b->ev_copy[s]) LBG_CUDA(cudaEventCreateWithFlags(&b->ev_copy[s], cudaEventDisableTiming));
            if (!b->ev_done[s]) LBG_CUDA(cudaEventCreateWithFlags(&b->ev_done[s], cudaEventDisableTiming));
            LBG_CUDA(cudaEventRecord(b->ev_done[s], b->stream));
        }
    }
    for (long long r0 = 0, c = 0; r0 < rows; r0 += chunk_rows, ++c) {
        const int s = (int)(c & 1);
        const long long nr = std::min(chunk_rows, rows - r0);
        const size_t bytes = sizeof(double) * (size_t)nr * w;
        const unsigned grid = (unsigned)((nr * w + 255) / 256);
        if (host_in) {
            LBG_CUDA(cudaStreamWaitEvent(b->side, b->ev_done[s], 0));
            LBG_CUDA(cudaMemcpyAsync(b->xfer[s], host_in + r0 * w, bytes, cudaMemcpyHostToDevice, b->side));
            LBG_CUDA(cudaEventRecord(b->ev_copy[s], b->side));
            LBG_CUDA(cudaStreamWaitEvent(b->stream, b->ev_copy[s], 0));
            repitch_kernel<<<grid, 256, 0, b->stream>>>(dev, b->xfer[s], nullptr, r0, nr, w, L.px);
            LBG_LAUNCH_CHECK();
            LBG_CUDA(cudaEventRecord(b->ev_done[s], b->stream));
        } else {
            LBG_CUDA(cudaStreamWaitEvent(b->stream, b->ev_done[s], 0));
            repitch_kernel<<<grid, 256, 0, b->stream>>>(dev, nullptr, b->xfer[s], r0, nr, w, L.px);
            LBG_LAUNCH_CHECK();
            LBG_CUDA(cudaEventRecord(b->ev_copy[s], b->stream));
            LBG_CUDA(cudaStreamWaitEvent(b->side, b->ev_copy[s], 0));
            LBG_CUDA(cudaMemcpyAsync(host_out + r0 * w, b->xfer[s], bytes, cudaMemcpyDeviceToHost, b->side));
            LBG_CUDA(cudaEventRecord(b->ev_done[s], b->side));
        }
    }
    LBG_CUDA(cudaStreamSynchronize(b->side));
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

static lbg_status copy_pdf(lbg_block b, double* dev, const double* host_in, double* host_out) {
    const Layout& L = b->L;
    const size_t width = sizeof(double) * (L.nx + 2);
    const size_t height = (size_t)kQ * L.py * L.pz;
    double* d0 = dev + (kXOff - 1);
    LBG_CUDA(cudaSetDevice(b->device));
    cudaPointerAttributes attr{};
    const void* hp = host_in ? (const void*)host_in : (const void*)host_out;
    if (width * height > (64u << 20) && cudaPointerGetAttributes(&attr, hp) == cudaSuccess &&
        attr.type == cudaMemoryTypeHost)
        return copy_pdf_pinned(b, dev, host_in, host_out);
    cudaGetLastError();  // pageable pointers are not an error
    if (host_in) {
        LBG_CUDA(cudaMemcpy2DAsync(d0, sizeof(double) * L.px, host_in, width, width, height,
                                   cudaMemcpyHostToDevice, b->stream));
    } else {
        LBG_CUDA(cudaMemcpy2DAsync(host_out, width, d0, sizeof(double) * L.px, width, height,
                                   cudaMemcpyDeviceToHost, b->stream));
    }
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

lbg_status lbg_upload_src(lbg_block b, const double* host) {
    if (b && b->aa) {  // an AA block takes the double-buffer src as its state S0
        b->aa_phase = 0;
        b->aa_pending = false;
    }
    return copy_pdf(b, b->src(), host, nullptr);
}
lbg_status lbg_download_src(lbg_block b, double* host) {
    if (b && b->aa && b->aa_phase == 1) {  // S1: the S0 image (post-collision, unstreamed) first
        LBG_CUDA(cudaSetDevice(b->device));
        double* tmp = nullptr;
        const size_t bytes = sizeof(double) * (kQ * (size_t)b->L.plane + 128);
        LBG_CUDA(cudaMallocAsync(&tmp, bytes, b->stream));
        LBG_CUDA(cudaMemsetAsync(tmp, 0, bytes, b->stream));
        lbg_status s = aa_unstream(b, tmp);
        if (s == LBG_OK) s = copy_pdf(b, tmp, nullptr, host);
        cudaFreeAsync(tmp, b->stream);
        return s;
    }
    return copy_pdf(b, b->src(), nullptr, host);
}
lbg_status lbg_upload_dst(lbg_block b, const double* host) {
    if (lbg_status s_ = aa_refuse(b, "lbg_upload_dst")) return s_;
    return copy_pdf(b, b->dst(), host, nullptr);
}
lbg_status lbg_download_dst(lbg_block b, double* host) {
    if (lbg_status s_ = aa_refuse(b, "lbg_download_dst")) return s_;
    return copy_pdf(b, b->dst(), nullptr, host);
}

lbg_status lbg_set_periodic_wrap(lbg_block b, const int wrap[3]) {
    if (!b || !wrap) return set_error(LBG_INVALID, "null argument");
    for (int a = 0; a < 3; ++a) b->wrap[a] = wrap[a] != 0;
    return LBG_OK;
}

lbg_status lbg_swap(lbg_block b) {
    if (b->aa) {  // in place: the swap completes the AA step (state S0 <-> S1)
        if (b->aa_pending) b->aa_phase ^= 1;
        b->aa_pending = false;
        return LBG_OK;
    }
    b->cur ^= 1;
    return LBG_OK;
}

lbg_status lbg_fill_equilibrium(lbg_block b, double rho, const double u[3]) {
    if (b->aa) {  // writes the src state: S0
        b->aa_phase = 0;
        b->aa_pending = false;
    }
    Feq f;
    equilibrium_host(rho, u, f.v);
    const Layout& L = b->L;
    LBG_CUDA(cudaSetDevice(b->device));
    dim3 grid((L.nx + 127) / 128, L.ny, L.nz);
    fill_interior_kernel<<<grid, 128, 0, b->stream>>>(b->src(), L, f);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_init_shear_wave(lbg_block b, const int domain[3]) {
    if (b->aa) {  // writes the src state: S0
        b->aa_phase = 0;
        b->aa_pending = false;
    }
    const Layout& L = b->L;
    LBG_CUDA(cudaSetDevice(b->device));
    dim3 grid((L.nx + 127) / 128, L.ny, L.nz);
    shear_wave_kernel<<<grid, 128, 0, b->stream>>>(b->src(), L, b->lo[0], b->lo[1], b->lo[2], domain[0],
                                                   domain[1], domain[2]);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_fill_ghosts_src(lbg_block b, double v) {
    const Layout& L = b->L;
    LBG_CUDA(cudaSetDevice(b->device));
    dim3 grid((L.nx + 2 + 127) / 128, L.ny + 2, L.nz + 2);
    fill_ghosts_kernel<<<grid, 128, 0, b->stream>>>(b->src(), L, v);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_sync(lbg_block b, lbg_errors* out) {
    LBG_CUDA(cudaSetDevice(b->device));
    LBG_CUDA(cudaStreamSynchronize(b->side));
    LBG_CUDA(cudaMemcpyAsync(b->err_h, b->err_d, sizeof(DeviceErrors), cudaMemcpyDeviceToHost,
                             b->stream));
    LBG_CUDA(cudaMemsetAsync(b->err_d, 0, sizeof(DeviceErrors), b->stream));
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    const DeviceErrors e = *b->err_h;
    if (out) {
        out->unstable_cells = (long long)e.unstable;
        out->overfull_cells = (long long)e.overfull;
        out->unknown_ids = (long long)e.unknown;
    }
    if (e.oob > 0)
        return set_error(LBG_CUDA_ERROR, "checked build: " + std::to_string(e.oob) +
                                             " out-of-range buffer indices (accesses skipped)");
    if (e.race > 0)
        return set_error(LBG_CUDA_ERROR, "checked build: " + std::to_string(e.race) +
                                             " cells written other than exactly once by a sweep");
    if (e.p2p_timeout > 0)
        return set_error(LBG_CUDA_ERROR, "P2P halo: neighbour did not publish its step (wait timed out)");
    if (e.overfull > 0)
        return set_error(LBG_NUMERIC_ERROR,
                         "more than two particles overlap a single cell in " +
                             std::to_string(e.overfull) +
                             " cells; particle penetration too deep for the coupling");
    if (e.unknown > 0)
        return set_error(LBG_SYNC_ERROR, "solid velocity field references " +
                                             std::to_string(e.unknown) +
                                             " unknown particle ids (ghost synchronization failed)");
    if (e.unstable > 0) {
        if (b->coupling)
            return set_error(LBG_NUMERIC_ERROR, "fluid instability in PSM kernel: " +
                                                    std::to_string(e.unstable) +
                                                    " cells out of range");
        return set_error(LBG_NUMERIC_ERROR, "fluid instability: " + std::to_string(e.unstable) +
                                                " cells with rho <= 0 or |u| > " +
                                                std::to_string(kMaxVelocity));
    }
    return LBG_OK;
}

static void nm_add_host(double& sum, double& comp, double v) {
    const double t = sum + v;
    if (std::fabs(sum) >= std::fabs(v))
        comp += (sum - t) + v;
    else
        comp += (v - t) + sum;
    sum = t;
}

static lbg_status moments(lbg_block b, double out[4]) {
    const Layout& L = b->L;
    const int rows = L.ny * L.nz;
    LBG_CUDA(cudaSetDevice(b->device));
    double* d = nullptr;
    LBG_CUDA(cudaMallocAsync(&d, sizeof(double) * 8 * rows, b->stream));
    row_moments_kernel<<<(rows + 127) / 128, 128, 0, b->stream>>>(b->src(), L, d);
    ::lbg::count_launch();
    std::vector<double> h((size_t)8 * rows);
    cudaError_t e = cudaMemcpyAsync(h.data(), d, sizeof(double) * 8 * rows, cudaMemcpyDeviceToHost,
                                    b->stream);
    cudaFreeAsync(d, b->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(b->stream);
    if (e != cudaSuccess) return cuda_check(e, "moments");
    for (int a = 0; a < 4; ++a) {
        double s = 0.0, c = 0.0;
        for (int r = 0; r < rows; ++r) {
            nm_add_host(s, c, h[(size_t)r * 8 + 2 * a]);
            c += h[(size_t)r * 8 + 2 * a + 1];
        }
        out[a] = s + c;
    }
    return LBG_OK;
}

lbg_status lbg_total_mass(lbg_block b, double* out) {
    if (lbg_status s_ = aa_refuse(b, "lbg_total_mass", true)) return s_;
    double m[4];
    lbg_status s = moments(b, m);
    if (s == LBG_OK) *out = m[0];
    return s;
}

lbg_status lbg_total_momentum(lbg_block b, double out[3]) {
    if (lbg_status s_ = aa_refuse(b, "lbg_total_momentum", true)) return s_;
    double m[4];
    lbg_status s = moments(b, m);
    if (s == LBG_OK)
        for (int a = 0; a < 3; ++a) out[a] = m[1 + a];
    return s;
}

lbg_status lbg_set_timing(lbg_block b, int on) {
    b->timing = on != 0;
    return LBG_OK;
}

lbg_status lbg_timings(lbg_block b, double ms[LBG_NUM_CATS], long long launches[LBG_NUM_CATS]) {
    LBG_CUDA(cudaSetDevice(b->device));
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    for (auto& s : b->spans) {
        float t = 0.f;
        LBG_CUDA(cudaEventElapsedTime(&t, s.a, s.b));
        b->acc_ms[s.cat] += t;
        b->acc_n[s.cat] += 1;
        b->event_pool.push_back(s.a);
        b->event_pool.push_back(s.b);
    }
    b->spans.clear();
    for (int c = 0; c < LBG_NUM_CATS; ++c) {
        if (ms) ms[c] = b->acc_ms[c];
        if (launches) launches[c] = b->acc_n[c];
        b->acc_ms[c] = 0.0;
        b->acc_n[c] = 0;
    }
    return LBG_OK;
}

}  // extern "C"
