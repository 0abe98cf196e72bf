// SPDX-License-Identifier: Apache-2.0
//
// K7 — PDF halo exchange of a slab decomposition over NCCL
//   reference: Simulation::begin_halo_exchange / complete_halo_exchange (sim.cpp:156-201),
//              source_slab / ghost_region (sim.cpp:120-152), PdfSlab (partition.hpp:77-81)
//
// The reference ships all 19 q of every boundary slab (faces, edges, corners) through the
// in-process MessageBus. A pull sweep only ever reads, from the ghost plane normal to the
// slab axis, the 5 populations whose velocity points into the block, so each face message
// here is 5 q x (interior face cells) doubles: 10.5 MB per direction at 512^2 instead of
// 39.8 MB. Edge ghosts of the received plane are produced by wrapping that plane locally
// along the other (periodic) axes — the same values the reference's edge messages carry.
//
//   begin:    event(compute) -> comm stream: pack kernel -> ncclGroup{Send/Recv x2}
//   complete: comm stream: unpack kernel (+ ring wrap) -> event -> compute stream waits
// The comm stream has the highest priority, so the NCCL kernels interleave with the inner
// sweep (the paper's communication hiding). With one rank and a periodic
// axis the exchange degenerates to a local wrap (no NCCL).
#include <nccl.h>

#include <cstring>

#include "lbg_internal.cuh"

namespace lbg {

struct Comm {
    ncclComm_t nccl = nullptr;
    int nranks = 1, rank = 0, axis = 2, periodic = 1;
    int prev = -1, next = -1;
    int na = 0, nb = 0;  // face extents (other two axes, a fastest)
    long long face = 0;  // na * nb
    double* send_lo = nullptr;  // plane 0,   q with c_axis = -1 -> prev
    double* send_hi = nullptr;  // plane n-1, q with c_axis = +1 -> next
    double* recv_lo = nullptr;  // from prev -> ghost plane -1,  q with c_axis = +1
    double* recv_hi = nullptr;  // from next -> ghost plane n,   q with c_axis = -1
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_src = nullptr, ev_done = nullptr, ev_t0 = nullptr;
    bool pending = false;
    int wrap_a = 0, wrap_b = 0;
    int q_up[5], q_dn[5];
};

__host__ __device__ inline int comp(int q, int axis) { return axis == 0 ? cx(q) : (axis == 1 ? cy(q) : cz(q)); }

struct HaloArgs {
    double* __restrict__ src;
    Layout L;
    int axis;
    int na, nb;
    int q_up[5], q_dn[5];
    const double* __restrict__ in_lo;
    const double* __restrict__ in_hi;
    double* __restrict__ out_lo;
    double* __restrict__ out_hi;
    int has_lo, has_hi;
    int wrap_a, wrap_b;  // periodic along the face axes
};

__device__ __forceinline__ long long cell3(const HaloArgs& h, int c_axis, int a, int b) {
    int ijk[3];
    const int ax = h.axis, aa = (ax + 1) % 3, ab = (ax + 2) % 3;
    ijk[ax] = c_axis;
    // face axes ordered so that `a` is the lower-index (faster) one
    const int fa = aa < ab ? aa : ab, fb = aa < ab ? ab : aa;
    ijk[fa] = a;
    ijk[fb] = b;
    return h.L.idx(ijk[0], ijk[1], ijk[2]);
}

__global__ void __launch_bounds__(256) halo_pack_kernel(const HaloArgs h) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long face = (long long)h.na * h.nb;
    if (t >= face) return;
    const int a = (int)(t % h.na), b = (int)(t / h.na);
    const int n_axis = h.axis == 0 ? h.L.nx : (h.axis == 1 ? h.L.ny : h.L.nz);
    const long long lo = cell3(h, 0, a, b), hi = cell3(h, n_axis - 1, a, b);
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        h.out_lo[s * face + t] = h.src[h.q_dn[s] * h.L.plane + lo];
        h.out_hi[s * face + t] = h.src[h.q_up[s] * h.L.plane + hi];
    }
}

// ghost planes incl. their ring: (a, b) in [-1, na] x [-1, nb]
__global__ void __launch_bounds__(256) halo_unpack_kernel(const HaloArgs h) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long ring = (long long)(h.na + 2) * (h.nb + 2);
    if (t >= ring) return;
    const int a = (int)(t % (h.na + 2)) - 1, b = (int)(t / (h.na + 2)) - 1;
    int sa = a, sb = b;
    if (a < 0 || a >= h.na) {
        if (!h.wrap_a) return;
        sa = a < 0 ? h.na - 1 : 0;
    }
    if (b < 0 || b >= h.nb) {
        if (!h.wrap_b) return;
        sb = b < 0 ? h.nb - 1 : 0;
    }
    const long long face = (long long)h.na * h.nb;
    const long long sidx = (long long)sb * h.na + sa;
    const int n_axis = h.axis == 0 ? h.L.nx : (h.axis == 1 ? h.L.ny : h.L.nz);
    if (h.has_lo) {
        const long long g = cell3(h, -1, a, b);
#pragma unroll
        for (int s = 0; s < 5; ++s) h.src[h.q_up[s] * h.L.plane + g] = h.in_lo[s * face + sidx];
    }
    if (h.has_hi) {
        const long long g = cell3(h, n_axis, a, b);
#pragma unroll
        for (int s = 0; s < 5; ++s) h.src[h.q_dn[s] * h.L.plane + g] = h.in_hi[s * face + sidx];
    }
}

// generic slab copy between the src buffer and a packed [q][k][j][i] buffer
__global__ void __launch_bounds__(256) slab_copy_kernel(double* __restrict__ src, Layout L, int lo0, int lo1,
                                                        int lo2, int e0, int e1, int e2,
                                                        double* __restrict__ buf, int to_buf) {
    const long long cells = (long long)e0 * e1 * e2;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cells * kQ) return;
    const int q = (int)(t / cells);
    const long long r = t % cells;
    const int i = lo0 + (int)(r % e0), j = lo1 + (int)((r / e0) % e1), k = lo2 + (int)(r / ((long long)e0 * e1));
    double* p = src + q * L.plane + L.idx(i, j, k);
    if (to_buf)
        buf[t] = *p;
    else
        *p = buf[t];
}

// all source slabs of a block in one launch (lbg_halo_stage): slab t covers the threads
// [begin[t], begin[t+1]) and is packed [q][k][j][i] into its own staging buffer, exactly as
// slab_copy_kernel(to_buf = 1) packs it
struct StageArgs {
    int n;
    int lo[26][3];
    int ext[26][3];
    long long begin[27];
    double* out[26];
};

__global__ void __launch_bounds__(256) slab_stage_kernel(const double* __restrict__ src, Layout L, StageArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.begin[a.n]) return;
    int s = 0;
    while (t >= a.begin[s + 1]) ++s;
    const long long u = t - a.begin[s];
    const long long cells = (long long)a.ext[s][0] * a.ext[s][1] * a.ext[s][2];
    const int q = (int)(u / cells);
    const long long r = u - q * cells;
    const int i = a.lo[s][0] + (int)(r % a.ext[s][0]);
    const int j = a.lo[s][1] + (int)((r / a.ext[s][0]) % a.ext[s][1]);
    const int k = a.lo[s][2] + (int)(r / ((long long)a.ext[s][0] * a.ext[s][1]));
    a.out[s][u] = src[q * L.plane + L.idx(i, j, k)];
}

// the receive side in one launch (lbg_halo_fetch_all): slab t is unpacked from out[t] into
// dst's ghost_region, as slab_copy_kernel(to_buf = 0) unpacks it
__global__ void __launch_bounds__(256) slab_unpack_kernel(double* __restrict__ src, Layout L, StageArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.begin[a.n]) return;
    int s = 0;
    while (t >= a.begin[s + 1]) ++s;
    const long long u = t - a.begin[s];
    const long long cells = (long long)a.ext[s][0] * a.ext[s][1] * a.ext[s][2];
    const int q = (int)(u / cells);
    const long long r = u - q * cells;
    const int i = a.lo[s][0] + (int)(r % a.ext[s][0]);
    const int j = a.lo[s][1] + (int)((r / a.ext[s][0]) % a.ext[s][1]);
    const int k = a.lo[s][2] + (int)(r / ((long long)a.ext[s][0] * a.ext[s][1]));
    src[q * L.plane + L.idx(i, j, k)] = a.out[s][u];
}

static lbg_status nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return LBG_OK;
    return set_error(LBG_CUDA_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}

static HaloArgs halo_args(lbg_block b) {
    Comm& c = *b->comm;
    HaloArgs h{};
    h.src = b->src();
    h.L = b->L;
    h.axis = c.axis;
    h.na = c.na;
    h.nb = c.nb;
    for (int s = 0; s < 5; ++s) {
        h.q_up[s] = c.q_up[s];
        h.q_dn[s] = c.q_dn[s];
    }
    return h;
}

}  // namespace lbg

using namespace lbg;

extern "C" {

lbg_status lbg_comm_unique_id(char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    if (lbg_status s = nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId")) return s;
    std::memcpy(out, &id, 128);
    return LBG_OK;
}

lbg_status lbg_comm_init(lbg_block b, int nranks, int rank, const char id[128], int axis,
                         const int periodic[3]) {
    if (lbg_status s_ = aa_refuse(b, "lbg_comm_init")) return s_;
    if (!b) return set_error(LBG_INVALID, "null block");
    if (axis < 0 || axis > 2 || nranks < 1 || rank < 0 || rank >= nranks)
        return set_error(LBG_INVALID, "bad comm arguments");
    if (b->comm) lbg_comm_destroy(b);
    LBG_CUDA(cudaSetDevice(b->device));
    auto* c = new Comm;
    b->comm = c;
    c->nranks = nranks;
    c->rank = rank;
    c->axis = axis;
    c->periodic = periodic[axis] != 0;
    c->prev = rank > 0 ? rank - 1 : (c->periodic ? nranks - 1 : -1);
    c->next = rank < nranks - 1 ? rank + 1 : (c->periodic ? 0 : -1);
    const int n[3] = {b->L.nx, b->L.ny, b->L.nz};
    const int aa = (axis + 1) % 3, ab = (axis + 2) % 3;
    c->na = n[aa < ab ? aa : ab];
    c->nb = n[aa < ab ? ab : aa];
    c->wrap_a = periodic[aa < ab ? aa : ab] != 0;
    c->wrap_b = periodic[aa < ab ? ab : aa] != 0;
    c->face = (long long)c->na * c->nb;
    int nu = 0, nd = 0;
    for (int q = 0; q < kQ; ++q) {
        if (comp(q, axis) == 1) c->q_up[nu++] = q;
        if (comp(q, axis) == -1) c->q_dn[nd++] = q;
    }
    const size_t bytes = sizeof(double) * 5 * c->face;
    LBG_CUDA(cudaMalloc(&c->send_lo, bytes));
    LBG_CUDA(cudaMalloc(&c->send_hi, bytes));
    LBG_CUDA(cudaMalloc(&c->recv_lo, bytes));
    LBG_CUDA(cudaMalloc(&c->recv_hi, bytes));
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    LBG_CUDA(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi_prio));
    LBG_CUDA(cudaEventCreateWithFlags(&c->ev_src, cudaEventDisableTiming));
    LBG_CUDA(cudaEventCreate(&c->ev_done));
    LBG_CUDA(cudaEventCreate(&c->ev_t0));
    if (nranks > 1) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        if (lbg_status s = nccl_check(ncclCommInitRank(&c->nccl, nranks, uid, rank), "ncclCommInitRank"))
            return s;
    }
    return LBG_OK;
}

}  // extern "C"

namespace lbg {
// the slab axis of the block's NCCL halo, -1 without lbg_comm_init (the host job's seam exchange)
int comm_axis(lbg_block b) { return (b && b->comm) ? b->comm->axis : -1; }
}  // namespace lbg

extern "C" {

lbg_status lbg_comm_destroy(lbg_block b) {
    if (!b || !b->comm) return LBG_OK;
    Comm* c = b->comm;
    cudaSetDevice(b->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->nccl) ncclCommDestroy(c->nccl);
    for (double* p : {c->send_lo, c->send_hi, c->recv_lo, c->recv_hi})
        if (p) cudaFree(p);
    if (c->ev_src) cudaEventDestroy(c->ev_src);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    if (c->ev_t0) cudaEventDestroy(c->ev_t0);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    b->comm = nullptr;
    return LBG_OK;
}

lbg_status lbg_halo_begin(lbg_block b) {
    if (!b || !b->comm) return set_error(LBG_INVALID, "halo exchange without lbg_comm_init");
    Comm& c = *b->comm;
    LBG_CUDA(cudaSetDevice(b->device));
    LBG_CUDA(cudaEventRecord(c.ev_src, b->stream));
    LBG_CUDA(cudaStreamWaitEvent(c.stream, c.ev_src, 0));
    LBG_CUDA(cudaEventRecord(c.ev_t0, c.stream));
    HaloArgs h = halo_args(b);
    h.out_lo = c.send_lo;
    h.out_hi = c.send_hi;
    halo_pack_kernel<<<(unsigned)((c.face + 255) / 256), 256, 0, c.stream>>>(h);
    LBG_LAUNCH_CHECK();
    if (c.nranks > 1) {
        const size_t cnt = 5 * (size_t)c.face;
        ncclGroupStart();
        // fixed posting order so the two messages between a rank pair match even when
        // prev == next (2 ranks, periodic): first up (hi -> next, lo <- prev), then down.
        if (c.next >= 0) ncclSend(c.send_hi, cnt, ncclDouble, c.next, c.nccl, c.stream);
        if (c.prev >= 0) ncclRecv(c.recv_lo, cnt, ncclDouble, c.prev, c.nccl, c.stream);
        if (c.prev >= 0) ncclSend(c.send_lo, cnt, ncclDouble, c.prev, c.nccl, c.stream);
        if (c.next >= 0) ncclRecv(c.recv_hi, cnt, ncclDouble, c.next, c.nccl, c.stream);
        if (lbg_status s = nccl_check(ncclGroupEnd(), "halo send/recv")) return s;
    }
    c.pending = true;
    return LBG_OK;
}

lbg_status lbg_halo_complete(lbg_block b) {
    if (!b || !b->comm) return set_error(LBG_INVALID, "halo exchange without lbg_comm_init");
    Comm& c = *b->comm;
    if (!c.pending) return set_error(LBG_SYNC_ERROR, "halo completion without a pending exchange");
    LBG_CUDA(cudaSetDevice(b->device));
    HaloArgs h = halo_args(b);
    const bool single = c.nranks == 1;  // periodic self-exchange
    h.in_lo = single ? c.send_hi : c.recv_lo;
    h.in_hi = single ? c.send_lo : c.recv_hi;
    h.has_lo = c.prev >= 0;
    h.has_hi = c.next >= 0;
    // the ghost ring of a received plane wraps along the face axes that are periodic,
    // reproducing the reference's edge-neighbour slabs (partition.cpp:62-79)
    h.wrap_a = c.wrap_a;
    h.wrap_b = c.wrap_b;
    const long long ring = (long long)(c.na + 2) * (c.nb + 2);
    halo_unpack_kernel<<<(unsigned)((ring + 255) / 256), 256, 0, c.stream>>>(h);
    LBG_LAUNCH_CHECK();
    LBG_CUDA(cudaEventRecord(c.ev_done, c.stream));
    LBG_CUDA(cudaStreamWaitEvent(b->stream, c.ev_done, 0));
    if (b->timing) {
        float ms = 0.f;
        // comm-stream span begin -> unpack done (synchronizes only when timing is on)
        LBG_CUDA(cudaEventSynchronize(c.ev_done));
        if (cudaEventElapsedTime(&ms, c.ev_t0, c.ev_done) == cudaSuccess) {
            b->acc_ms[LBG_CAT_PSM_COMM] += ms;
            b->acc_n[LBG_CAT_PSM_COMM] += 1;
        }
    }
    c.pending = false;
    return LBG_OK;
}

}  // extern "C"

namespace {

// source_slab (sim.cpp:120-135) for pack, ghost_region (sim.cpp:137-152) for unpack
void slab_box(const lbg::Layout& L, const int off[3], bool ghost, int lo[3], int ext[3]) {
    const int n[3] = {L.nx, L.ny, L.nz};
    for (int a = 0; a < 3; ++a) {
        if (off[a] == 1) {
            lo[a] = ghost ? n[a] : n[a] - 1;
            ext[a] = 1;
        } else if (off[a] == -1) {
            lo[a] = ghost ? -1 : 0;
            ext[a] = 1;
        } else {
            lo[a] = 0;
            ext[a] = n[a];
        }
    }
}

lbg_status slab_io(lbg_block b, const int off[3], bool ghost, double* host, long long capacity,
                   long long* n_out, bool to_host) {
    using namespace lbg;
    if (!b || !off || !host) return set_error(LBG_INVALID, "null argument");
    int lo[3], ext[3];
    slab_box(b->L, off, ghost, lo, ext);
    const long long n = (long long)kQ * ext[0] * ext[1] * ext[2];
    if (n_out) *n_out = n;
    if (capacity < n) return set_error(LBG_INVALID, "slab buffer too small");
    LBG_CUDA(cudaSetDevice(b->device));
    double* d = nullptr;
    LBG_CUDA(cudaMallocAsync(&d, sizeof(double) * n, b->stream));
    if (!to_host) LBG_CUDA(cudaMemcpyAsync(d, host, sizeof(double) * n, cudaMemcpyHostToDevice, b->stream));
    slab_copy_kernel<<<(unsigned)((n + 255) / 256), 256, 0, b->stream>>>(b->src(), b->L, lo[0], lo[1], lo[2],
                                                                         ext[0], ext[1], ext[2], d, to_host);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && to_host)
        e = cudaMemcpyAsync(host, d, sizeof(double) * n, cudaMemcpyDeviceToHost, b->stream);
    cudaFreeAsync(d, b->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(b->stream);
    if (e != cudaSuccess) return cuda_check(e, "slab copy");
    return LBG_OK;
}

// after dst's unpack of the staged slabs of `srcs`: record dst's stream position and register
// it with every source, whose next lbg_halo_stage waits for it
lbg_status note_consumed(lbg_block dst, const lbg_block* srcs, int n) {
    using namespace lbg;
    if (!dst->ev_fetched) LBG_CUDA(cudaEventCreateWithFlags(&dst->ev_fetched, cudaEventDisableTiming));
    LBG_CUDA(cudaEventRecord(dst->ev_fetched, dst->stream));
    for (int t = 0; t < n; ++t) {
        lbg_block s = srcs[t];
        std::lock_guard<std::mutex> g(s->consumers_mu);
        bool have = false;
        for (cudaEvent_t e : s->consumers) have = have || e == dst->ev_fetched;
        if (!have) s->consumers.push_back(dst->ev_fetched);
    }
    return LBG_OK;
}

}  // namespace

extern "C" {

lbg_status lbg_pack_slab(lbg_block b, const int off[3], double* out, long long capacity, long long* n_out) {
    if (lbg_status s_ = aa_refuse(b, "lbg_pack_slab")) return s_;
    return slab_io(b, off, false, out, capacity, n_out, true);
}

lbg_status lbg_unpack_slab(lbg_block b, const int dir[3], const double* in, long long n) {
    if (lbg_status s_ = aa_refuse(b, "lbg_unpack_slab")) return s_;
    return slab_io(b, dir, true, const_cast<double*>(in), n, nullptr, false);
}

lbg_status lbg_halo_stage(lbg_block b, const int (*offs)[3], int n) {
    if (lbg_status s_ = aa_refuse(b, "lbg_halo_stage")) return s_;
    using namespace lbg;
    if (!b || (n > 0 && !offs)) return set_error(LBG_INVALID, "null argument");
    LBG_CUDA(cudaSetDevice(b->device));
    if (!b->ev_stage) LBG_CUDA(cudaEventCreateWithFlags(&b->ev_stage, cudaEventDisableTiming));
    if (n > 26) return set_error(LBG_INVALID, "at most 26 halo neighbours");
    Span span(b, LBG_CAT_PSM_COMM);
    {
        // the receivers of the previous staging have unpacked it (stream order, any device)
        std::lock_guard<std::mutex> g(b->consumers_mu);
        for (cudaEvent_t e : b->consumers) LBG_CUDA(cudaStreamWaitEvent(b->stream, e, 0));
        b->consumers.clear();
    }
    StageArgs a{};
    a.n = 0;
    a.begin[0] = 0;
    for (int t = 0; t < n; ++t) {
        int lo[3], ext[3];
        slab_box(b->L, offs[t], false, lo, ext);
        const size_t cnt = (size_t)kQ * ext[0] * ext[1] * ext[2];
        const int key = (offs[t][0] + 1) * 9 + (offs[t][1] + 1) * 3 + (offs[t][2] + 1);
        if (lbg_status s = grow_device(b->stage[key], b->stage_cap[key], (long long)cnt, (long long)cnt,
                                       "cudaMalloc(halo staging)"))
            return s;
        for (int c = 0; c < 3; ++c) {
            a.lo[a.n][c] = lo[c];
            a.ext[a.n][c] = ext[c];
        }
        a.out[a.n] = b->stage[key];
        a.begin[a.n + 1] = a.begin[a.n] + (long long)cnt;
        ++a.n;
    }
    if (a.n > 0) {  // every neighbour's slab in one launch
        slab_stage_kernel<<<(unsigned)((a.begin[a.n] + 255) / 256), 256, 0, b->stream>>>(b->src(), b->L, a);
        LBG_LAUNCH_CHECK();
    }
    LBG_CUDA(cudaEventRecord(b->ev_stage, b->stream));
    return LBG_OK;
}

lbg_status lbg_halo_fetch(lbg_block dst, const int dir[3], lbg_block src) {
    using namespace lbg;
    if (!dst || !src || !dir) return set_error(LBG_INVALID, "null argument");
    const int back[3] = {-dir[0], -dir[1], -dir[2]};
    const int key = (back[0] + 1) * 9 + (back[1] + 1) * 3 + (back[2] + 1);
    int lo[3], ext[3];
    slab_box(dst->L, dir, true, lo, ext);
    const size_t cnt = (size_t)kQ * ext[0] * ext[1] * ext[2];
    if (!src->stage[key] || src->stage_cap[key] < cnt)
        return set_error(LBG_SYNC_ERROR, "halo completion without a pending exchange");
    LBG_CUDA(cudaSetDevice(dst->device));
    Span span(dst, LBG_CAT_PSM_COMM);
    LBG_CUDA(cudaStreamWaitEvent(dst->stream, src->ev_stage, 0));
    const double* from = src->stage[key];
    if (src->device != dst->device) {
        if (lbg_status s = grow_device(dst->recv_buf, dst->recv_cap, (long long)cnt, (long long)cnt,
                                       "cudaMalloc(halo receive)"))
            return s;
        LBG_CUDA(cudaMemcpyPeerAsync(dst->recv_buf, dst->device, from, src->device, sizeof(double) * cnt,
                                     dst->stream));
        from = dst->recv_buf;
    }
    slab_copy_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, dst->stream>>>(
        dst->src(), dst->L, lo[0], lo[1], lo[2], ext[0], ext[1], ext[2], const_cast<double*>(from), 0);
    LBG_LAUNCH_CHECK();
    return note_consumed(dst, &src, 1);
}

lbg_status lbg_halo_fetch_all(lbg_block dst, const int (*dirs)[3], const lbg_block* srcs, int n) {
    using namespace lbg;
    if (!dst || (n > 0 && (!dirs || !srcs))) return set_error(LBG_INVALID, "null argument");
    if (n > 26) return set_error(LBG_INVALID, "at most 26 halo neighbours");
    LBG_CUDA(cudaSetDevice(dst->device));
    Span span(dst, LBG_CAT_PSM_COMM);
    StageArgs a{};
    a.begin[0] = 0;
    for (int t = 0; t < n; ++t) {
        lbg_block src = srcs[t];
        if (!src) return set_error(LBG_INVALID, "null source block");
        const int back[3] = {-dirs[t][0], -dirs[t][1], -dirs[t][2]};
        const int key = (back[0] + 1) * 9 + (back[1] + 1) * 3 + (back[2] + 1);
        int lo[3], ext[3];
        slab_box(dst->L, dirs[t], true, lo, ext);
        const size_t cnt = (size_t)kQ * ext[0] * ext[1] * ext[2];
        if (!src->stage[key] || src->stage_cap[key] < cnt)
            return set_error(LBG_SYNC_ERROR, "halo completion without a pending exchange");
        LBG_CUDA(cudaStreamWaitEvent(dst->stream, src->ev_stage, 0));
        const double* from = src->stage[key];
        if (src->device != dst->device) {  // NVLink peer copy into this block's receive slot
            const int rkey = (dirs[t][0] + 1) * 9 + (dirs[t][1] + 1) * 3 + (dirs[t][2] + 1);
            if (lbg_status st = grow_device(dst->recv_multi[rkey], dst->recv_multi_cap[rkey], (long long)cnt,
                                            (long long)cnt, "cudaMalloc(halo receive)"))
                return st;
            LBG_CUDA(cudaMemcpyPeerAsync(dst->recv_multi[rkey], dst->device, from, src->device,
                                         sizeof(double) * cnt, dst->stream));
            from = dst->recv_multi[rkey];
        }
        for (int c = 0; c < 3; ++c) {
            a.lo[a.n][c] = lo[c];
            a.ext[a.n][c] = ext[c];
        }
        a.out[a.n] = const_cast<double*>(from);
        a.begin[a.n + 1] = a.begin[a.n] + (long long)cnt;
        ++a.n;
    }
    if (a.n > 0) {  // every neighbour's slab in one launch
        slab_unpack_kernel<<<(unsigned)((a.begin[a.n] + 255) / 256), 256, 0, dst->stream>>>(dst->src(), dst->L, a);
        LBG_LAUNCH_CHECK();
    }
    return note_consumed(dst, srcs, n);
}

}  // extern "C"
