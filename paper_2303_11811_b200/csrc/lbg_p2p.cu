// SPDX-License-Identifier: Apache-2.0
//
// K7' — the slab halo fused into the outer sweep over NVLink peer memory.
//   reference: begin/complete_halo_exchange (sim.cpp:156-201) + the outer run_kernel
//   (sim.cpp:315) for a {1,1,N} / {N,1,1} block grid, one block (process) per GPU.
//
// Instead of pack -> NCCL send/recv -> unpack, the kernel that computes a rank's two
// boundary planes stores the 5 populations leaving through each face straight into the
// neighbour GPU's ghost plane (remote stores through the CUDA-IPC-mapped PDF buffer, coalesced
// rows, NVLink 5), so the transfer overlaps the collision math tile by tile and no
// separate communication kernel or staging buffer exists. Both ranks swap buffers in lockstep,
// so the neighbour's next-step source buffer is buf[cur ^ 1] on both sides.
//
// Ordering: the last CTA of the outer sweep publishes `step + 1` into the neighbours' flag
// words (system-scope release after a system fence). Before its next outer sweep a rank waits
// (one-thread kernel, acquire loads, bounded spin) until both neighbours have published the
// step, which is exactly when (a) their writes into this rank's ghost planes have landed and
// (b) they have finished reading the ghost planes this rank is about to overwrite. The inner
// sweep (slab-axis planes 1..n-2) needs no ghost and runs before the wait, so the wait is
// normally already satisfied. One rank per GPU only (the waits are cross-GPU).
#include <cstring>

#include "lbg_cell.cuh"
#include "lbg_internal.cuh"

namespace lbg {

struct P2P {
    int nranks = 1, rank = 0, axis = 2;
    int prev = -1, next = -1;
    int wrap_face[2] = {0, 0};  // face axes (lower index first) periodic
    double* rbuf_prev[2] = {nullptr, nullptr};
    double* rbuf_next[2] = {nullptr, nullptr};
    unsigned long long* rflag_prev = nullptr;  // prev's flag words
    unsigned long long* rflag_next = nullptr;
    unsigned long long* flags = nullptr;  // mine: [0] published by prev, [1] by next, [2] CTA counter
    void* opened[6] = {};
    int n_opened = 0;
    unsigned long long step = 0;
};

struct OuterArgs {
    const double* __restrict__ src;
    double* __restrict__ dst;
    Layout L;
    double inv_tau;
    Force F;
    DeviceErrors* err;
    int wrap[3];
    int axis, na, nb;
    double* rprev;  // neighbour dst buffers (remote)
    double* rnext;
    unsigned long long* rflag_prev;
    unsigned long long* rflag_next;
    unsigned long long* ctr;
    unsigned long long publish;
    int q_up[5], q_dn[5];
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <bool kForced>
__global__ void __launch_bounds__(256) outer_p2p_kernel(const OuterArgs a) {
    const long long face = (long long)a.na * a.nb;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool ok = true;
    if (t < 2 * face) {
        const int side = (int)(t / face);  // 0: plane 0 (-> prev), 1: plane n-1 (-> next)
        const long long r = t % face;
        const int fa = (int)(r % a.na), fb = (int)(r / a.na);
        const int n_axis = a.axis == 0 ? a.L.nx : (a.axis == 1 ? a.L.ny : a.L.nz);
        int ijk[3];
        const int aa = (a.axis + 1) % 3, ab = (a.axis + 2) % 3;
        const int lo_ax = aa < ab ? aa : ab, hi_ax = aa < ab ? ab : aa;
        ijk[a.axis] = side == 0 ? 0 : n_axis - 1;
        ijk[lo_ax] = fa;
        ijk[hi_ax] = fb;
        const Layout& L = a.L;
        const long long base = L.idx(ijk[0], ijk[1], ijk[2]);
        // pull with the face axes wrapped in-kernel; slab-axis ghosts were written by the peer
        const long long sy = L.px, sz = (long long)L.px * L.py;
        const long long xl = (a.wrap[0] && ijk[0] == 0) ? L.nx : 0;
        const long long xh = (a.wrap[0] && ijk[0] == L.nx - 1) ? -(long long)L.nx : 0;
        const long long yl = (a.wrap[1] && ijk[1] == 0) ? L.ny * sy : 0;
        const long long yh = (a.wrap[1] && ijk[1] == L.ny - 1) ? -L.ny * sy : 0;
        const long long zl = (a.wrap[2] && ijk[2] == 0) ? L.nz * sz : 0;
        const long long zh = (a.wrap[2] && ijk[2] == L.nz - 1) ? -L.nz * sz : 0;
        double f[kQ];
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const long long corr = (cx(q) == 1 ? xl : (cx(q) == -1 ? xh : 0)) +
                                   (cy(q) == 1 ? yl : (cy(q) == -1 ? yh : 0)) +
                                   (cz(q) == 1 ? zl : (cz(q) == -1 ? zh : 0));
            f[q] = a.src[q * L.plane + base - L.shift(q) + corr];
        }
        ok = srt_cell<kForced>(f, a.inv_tau, a.F);
#pragma unroll
        for (int q = 0; q < kQ; ++q) a.dst[q * L.plane + base] = f[q];
        // the populations leaving through this face -> the neighbour's ghost plane
        int g[3] = {ijk[0], ijk[1], ijk[2]};
        g[a.axis] = side == 0 ? n_axis : -1;
        const long long gi = L.idx(g[0], g[1], g[2]);
        double* remote = side == 0 ? a.rprev : a.rnext;
        if (remote) {
#pragma unroll
            for (int s = 0; s < 5; ++s) {
                const int q = side == 0 ? a.q_dn[s] : a.q_up[s];
                double v = 0.0;
#pragma unroll
                for (int qq = 0; qq < kQ; ++qq)
                    if (qq == q) v = f[qq];
                remote[q * L.plane + gi] = v;
            }
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, !ok);
    if (m && (threadIdx.x & 31) == 0) atomicAdd(&a.err->unstable, (unsigned long long)__popc(m));
    // last CTA publishes the step to both neighbours (CTA barrier, then one system fence by
    // the CTA's first thread: the grid-sync pattern, cumulative over the CTA's stores)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned long long done = atomicAdd(a.ctr, 1ull) + 1;
        if (done == gridDim.x) {
            *a.ctr = 0;
            __threadfence_system();
            if (a.rflag_prev) st_release_sys(a.rflag_prev + 1, a.publish);  // I am prev's next
            if (a.rflag_next) st_release_sys(a.rflag_next + 0, a.publish);  // I am next's prev
        }
    }
}

__global__ void p2p_wait_kernel(const unsigned long long* flags, int need_prev, int need_next,
                                unsigned long long step, DeviceErrors* err) {
    long long spins = 0;
    while ((need_prev && ld_acquire_sys(flags + 0) < step) || (need_next && ld_acquire_sys(flags + 1) < step)) {
        __nanosleep(200);
        if (++spins > 50000000LL) {  // ~10 s: report instead of hanging the GPU
            atomicAdd(&err->p2p_timeout, 1ull);
            return;
        }
    }
}

// one-time fill of this rank's slab-axis ghost planes from the neighbours' src boundary planes
__global__ void p2p_prime_kernel(double* __restrict__ src, Layout L, int axis, int na, int nb,
                                 const double* __restrict__ rprev, const double* __restrict__ rnext,
                                 int q_up0, int q_up1, int q_up2, int q_up3, int q_up4, int q_dn0, int q_dn1,
                                 int q_dn2, int q_dn3, int q_dn4) {
    const long long face = (long long)na * nb;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * face) return;
    const int side = (int)(t / face);
    const long long r = t % face;
    const int fa = (int)(r % na), fb = (int)(r / na);
    const int n_axis = axis == 0 ? L.nx : (axis == 1 ? L.ny : L.nz);
    const int aa = (axis + 1) % 3, ab = (axis + 2) % 3;
    const int lo_ax = aa < ab ? aa : ab, hi_ax = aa < ab ? ab : aa;
    int g[3], s[3];
    g[lo_ax] = s[lo_ax] = fa;
    g[hi_ax] = s[hi_ax] = fb;
    // side 0: my ghost -1 <- prev's plane n-1 (q_up); side 1: my ghost n <- next's plane 0 (q_dn)
    g[axis] = side == 0 ? -1 : n_axis;
    s[axis] = side == 0 ? n_axis - 1 : 0;
    const double* from = side == 0 ? rprev : rnext;
    if (!from) return;
    const int qs[5] = {side == 0 ? q_up0 : q_dn0, side == 0 ? q_up1 : q_dn1, side == 0 ? q_up2 : q_dn2,
                       side == 0 ? q_up3 : q_dn3, side == 0 ? q_up4 : q_dn4};
    const long long gi = L.idx(g[0], g[1], g[2]), si = L.idx(s[0], s[1], s[2]);
#pragma unroll
    for (int k = 0; k < 5; ++k) src[qs[k] * L.plane + gi] = from[qs[k] * L.plane + si];
}

static int axis_comp(int q, int axis) { return axis == 0 ? cx(q) : (axis == 1 ? cy(q) : cz(q)); }

}  // namespace lbg

using namespace lbg;

namespace {
constexpr size_t kHandle = sizeof(cudaIpcMemHandle_t);  // 64
// per rank: 3 IPC handles, then the block's device layout (nx, ny, nz, px) — the remote
// stores index the peer's PDF buffer with the local Layout, so every rank must match
constexpr size_t kRankBytes = 3 * kHandle + 4 * sizeof(int);

lbg_status ensure_p2p(lbg_block b) {
    if (!b->p2p) b->p2p = new P2P;
    if (!b->p2p->flags) {
        LBG_CUDA(cudaMalloc(&b->p2p->flags, 4 * sizeof(unsigned long long)));
        LBG_CUDA(cudaMemset(b->p2p->flags, 0, 4 * sizeof(unsigned long long)));
    }
    return LBG_OK;
}
}  // namespace

extern "C" {

lbg_status lbg_p2p_handles(lbg_block b, void* out, size_t* bytes) {
    if (!b || !out) return set_error(LBG_INVALID, "null argument");
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = ensure_p2p(b)) return s;
    char* o = static_cast<char*>(out);
    cudaIpcMemHandle_t h;
    LBG_CUDA(cudaIpcGetMemHandle(&h, b->buf[0]));
    std::memcpy(o, &h, kHandle);
    LBG_CUDA(cudaIpcGetMemHandle(&h, b->buf[1]));
    std::memcpy(o + kHandle, &h, kHandle);
    LBG_CUDA(cudaIpcGetMemHandle(&h, b->p2p->flags));
    std::memcpy(o + 2 * kHandle, &h, kHandle);
    const int geo[4] = {b->L.nx, b->L.ny, b->L.nz, b->L.px};
    std::memcpy(o + 3 * kHandle, geo, sizeof(geo));
    if (bytes) *bytes = kRankBytes;
    return LBG_OK;
}

lbg_status lbg_p2p_connect(lbg_block b, int nranks, int rank, const void* all, int axis, const int periodic[3]) {
    if (lbg_status s_ = aa_refuse(b, "lbg_p2p_connect")) return s_;
    if (!b || !all || !periodic) return set_error(LBG_INVALID, "null argument");
    if (axis < 0 || axis > 2 || nranks < 2 || rank < 0 || rank >= nranks)
        return set_error(LBG_INVALID, "p2p halo needs >= 2 ranks and a slab axis");
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = ensure_p2p(b)) return s;
    P2P& p = *b->p2p;
    p.nranks = nranks;
    p.rank = rank;
    p.axis = axis;
    p.prev = rank > 0 ? rank - 1 : (periodic[axis] ? nranks - 1 : -1);
    p.next = rank < nranks - 1 ? rank + 1 : (periodic[axis] ? 0 : -1);
    const char* h = static_cast<const char*>(all);
    for (int r : {p.prev, p.next}) {
        if (r < 0) continue;
        int geo[4];
        std::memcpy(geo, h + (size_t)r * kRankBytes + 3 * kHandle, sizeof(geo));
        if (geo[0] != b->L.nx || geo[1] != b->L.ny || geo[2] != b->L.nz || geo[3] != b->L.px)
            return set_error(LBG_INVALID, "p2p halo: neighbour block dimensions differ (equal slabs required)");
    }
    auto open = [&](int r, double* bufs[2], unsigned long long** flag) -> lbg_status {
        for (int s = 0; s < 2; ++s) {
            cudaIpcMemHandle_t mh;
            std::memcpy(&mh, h + (size_t)r * kRankBytes + s * kHandle, kHandle);
            void* ptr = nullptr;
            LBG_CUDA(cudaIpcOpenMemHandle(&ptr, mh, cudaIpcMemLazyEnablePeerAccess));
            bufs[s] = static_cast<double*>(ptr);
            p.opened[p.n_opened++] = ptr;
        }
        cudaIpcMemHandle_t mh;
        std::memcpy(&mh, h + (size_t)r * kRankBytes + 2 * kHandle, kHandle);
        void* ptr = nullptr;
        LBG_CUDA(cudaIpcOpenMemHandle(&ptr, mh, cudaIpcMemLazyEnablePeerAccess));
        *flag = static_cast<unsigned long long*>(ptr);
        p.opened[p.n_opened++] = ptr;
        return LBG_OK;
    };
    if (p.prev >= 0)
        if (lbg_status s = open(p.prev, p.rbuf_prev, &p.rflag_prev)) return s;
    if (p.next >= 0) {
        if (p.next == p.prev) {
            p.rbuf_next[0] = p.rbuf_prev[0];
            p.rbuf_next[1] = p.rbuf_prev[1];
            p.rflag_next = p.rflag_prev;
        } else if (lbg_status s = open(p.next, p.rbuf_next, &p.rflag_next)) {
            return s;
        }
    }
    p.step = 0;
    return LBG_OK;
}

lbg_status lbg_p2p_prime(lbg_block b) {
    if (!b || !b->p2p || b->p2p->nranks < 2) return set_error(LBG_INVALID, "lbg_p2p_connect first");
    P2P& p = *b->p2p;
    LBG_CUDA(cudaSetDevice(b->device));
    const int n[3] = {b->L.nx, b->L.ny, b->L.nz};
    const int aa = (p.axis + 1) % 3, ab = (p.axis + 2) % 3;
    const int na = n[aa < ab ? aa : ab], nb = n[aa < ab ? ab : aa];
    int up[5], dn[5], nu = 0, nd = 0;
    for (int q = 0; q < kQ; ++q) {
        if (axis_comp(q, p.axis) == 1) up[nu++] = q;
        if (axis_comp(q, p.axis) == -1) dn[nd++] = q;
    }
    const long long cnt = 2LL * na * nb;
    p2p_prime_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, b->stream>>>(
        b->src(), b->L, p.axis, na, nb, p.prev >= 0 ? p.rbuf_prev[b->cur] : nullptr,
        p.next >= 0 ? p.rbuf_next[b->cur] : nullptr, up[0], up[1], up[2], up[3], up[4], dn[0], dn[1], dn[2],
        dn[3], dn[4]);
    LBG_LAUNCH_CHECK();
    LBG_CUDA(cudaStreamSynchronize(b->stream));
    return LBG_OK;
}

lbg_status lbg_sweep_outer_p2p(lbg_block b, const lbg_fluid* fl) {
    if (!b || !fl) return set_error(LBG_INVALID, "null argument");
    if (!b->p2p || b->p2p->nranks < 2) return set_error(LBG_INVALID, "lbg_p2p_connect first");
    if (b->coupling) return set_error(LBG_INVALID, "the P2P outer sweep is the plain-fluid path");
    if (!(fl->tau > 0.5))
        return set_error(LBG_CONFIG_ERROR, "fluid relaxation time tau must be > 0.5 (got " +
                                               std::to_string(fl->tau) + ")");
    P2P& p = *b->p2p;
    LBG_CUDA(cudaSetDevice(b->device));
    const int n[3] = {b->L.nx, b->L.ny, b->L.nz};
    const int aa = (p.axis + 1) % 3, ab = (p.axis + 2) % 3;
    OuterArgs a{};
    a.src = b->src();
    a.dst = b->dst();
    a.L = b->L;
    a.inv_tau = 1.0 / fl->tau;
    a.F = {fl->f_ext[0], fl->f_ext[1], fl->f_ext[2]};
    a.err = b->err_d;
    for (int c = 0; c < 3; ++c) a.wrap[c] = b->wrap[c];
    a.wrap[p.axis] = 0;
    a.axis = p.axis;
    a.na = n[aa < ab ? aa : ab];
    a.nb = n[aa < ab ? ab : aa];
    a.rprev = p.prev >= 0 ? p.rbuf_prev[b->cur ^ 1] : nullptr;
    a.rnext = p.next >= 0 ? p.rbuf_next[b->cur ^ 1] : nullptr;
    a.rflag_prev = p.prev >= 0 ? p.rflag_prev : nullptr;
    a.rflag_next = p.next >= 0 ? p.rflag_next : nullptr;
    a.ctr = p.flags + 2;
    a.publish = p.step + 1;
    int nu = 0, nd = 0;
    for (int q = 0; q < kQ; ++q) {
        if (axis_comp(q, p.axis) == 1) a.q_up[nu++] = q;
        if (axis_comp(q, p.axis) == -1) a.q_dn[nd++] = q;
    }
    Span span(b, LBG_CAT_PSM);
    // neighbours finished the previous outer sweep: ghosts landed, old ghosts free to overwrite
    p2p_wait_kernel<<<1, 1, 0, b->stream>>>(p.flags, p.prev >= 0, p.next >= 0, p.step, b->err_d);
    LBG_LAUNCH_CHECK();
    const long long cells = 2LL * a.na * a.nb;
    const unsigned grid = (unsigned)((cells + 255) / 256);
    const bool forced = fl->f_ext[0] != 0.0 || fl->f_ext[1] != 0.0 || fl->f_ext[2] != 0.0;
    forced ? outer_p2p_kernel<true><<<grid, 256, 0, b->stream>>>(a)
           : outer_p2p_kernel<false><<<grid, 256, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
    p.step += 1;
    return LBG_OK;
}

lbg_status lbg_p2p_destroy(lbg_block b) {
    if (!b || !b->p2p) return LBG_OK;
    cudaSetDevice(b->device);
    cudaStreamSynchronize(b->stream);
    P2P& p = *b->p2p;
    for (int i = 0; i < p.n_opened; ++i) cudaIpcCloseMemHandle(p.opened[i]);
    if (p.flags) cudaFree(p.flags);
    delete b->p2p;
    b->p2p = nullptr;
    return LBG_OK;
}

}  // extern "C"
