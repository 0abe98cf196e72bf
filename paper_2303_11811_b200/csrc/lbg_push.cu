// SPDX-License-Identifier: Apache-2.0
//
// K7'' — the PDF halo pushed by its sender, for blocks of one process on any GPUs (the
// drop-in's block workers). Replaces begin/complete_halo_exchange (sim.cpp:156-201) after the
// first step.
//
// The reference ships all 19 q of each of the 26 boundary slabs to the neighbours and the
// receiver copies them into its ghost regions. A pull sweep only reads a ghost slot (g, q)
// when g + c_q is one of its interior cells, i.e. only the populations that stream out of the
// sender through that face (5 q per face cell) or edge (1 q per edge cell; D3Q19 has no corner
// velocities). So right after a block's sweep, lbg_halo_push copies exactly those post-collision
// values from its fresh dst buffer into each neighbour's dst buffer — the neighbour's source of
// the next step, after both swap — at the neighbour's ghost coordinates: one kernel per block
// and step, device stores straight into the neighbour's HBM (NVLink peer stores when it lives
// on another GPU), no staging buffer, no receiver-side copy or unpack. It runs on the block's
// comm stream and overlaps whatever the host does next (the DEM sub-cycles); the receiver's
// lbg_halo_push_wait orders its next step after the pushes it depends on. These are the values
// source_slab/ghost_region would have carried (the sender's dst after the sweep is its src after
// the swap), so every interior result is bitwise the reference's.
//
// Ordering: the push of step n writes the neighbour's buffer that the neighbour read as its
// source in step n-1, so it is issued after the neighbour's step n-1 sweep (the event recorded
// by that neighbour's last push). Events alternate by step parity so a receiver waiting for
// step n never races with its sender already recording step n+1.
#include <atomic>
#include <cstring>

#include "lbg_internal.cuh"

namespace lbg {

constexpr int kMaxPush = 26;

struct PushArgs {
    int n;
    int lo[kMaxPush][3];
    int ext[kMaxPush][3];
    int sh[kMaxPush][3];  // neighbour-local = local + sh
    int nq[kMaxPush];
    int q[kMaxPush][5];
    double* dst[kMaxPush];
    int px[kMaxPush], py[kMaxPush];
    long long plane[kMaxPush];
    long long begin[kMaxPush + 1];
    DeviceErrors* err;
};

struct Push {
    int n = 0;
    int off[kMaxPush][3];
    lbg_block nbr[kMaxPush];
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_swept = nullptr;
    cudaEvent_t ev_push[2] = {nullptr, nullptr};
    std::atomic<long long> count{0};  // pushes issued (read by the neighbours' threads)
};

__global__ void __launch_bounds__(256) halo_push_kernel(const double* __restrict__ src, Layout L, PushArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.begin[a.n]) return;
    int s = 0;
    while (t >= a.begin[s + 1]) ++s;
    // 32-bit index math within a slab (a face has < 2^31 cells)
    const unsigned u = (unsigned)(t - a.begin[s]);
    const unsigned cells = (unsigned)a.ext[s][0] * a.ext[s][1] * a.ext[s][2];
    const int qi = (int)(u / cells);
    const unsigned r = u - qi * cells, row = r / (unsigned)a.ext[s][0];
    const int i = a.lo[s][0] + (int)(r - row * (unsigned)a.ext[s][0]);
    const int j = a.lo[s][1] + (int)(row % (unsigned)a.ext[s][1]);
    const int k = a.lo[s][2] + (int)(row / (unsigned)a.ext[s][1]);
    const int q = a.q[s][qi];
    const double v = src[q * L.plane + LBG_IDX(L.idx(i, j, k), L.plane, a.err)];
    const long long bi = i + a.sh[s][0], bj = j + a.sh[s][1], bk = k + a.sh[s][2];
    a.dst[s][q * a.plane[s] + LBG_IDX(((bk + 1) * a.py[s] + (bj + 1)) * a.px[s] + kXOff + bi, a.plane[s], a.err)] = v;
}

}  // namespace lbg

using namespace lbg;

extern "C" {

lbg_status lbg_halo_push_destroy(lbg_block b) {
    if (!b || !b->push) return LBG_OK;
    Push* p = b->push;
    cudaSetDevice(b->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    if (p->ev_swept) cudaEventDestroy(p->ev_swept);
    for (auto e : p->ev_push)
        if (e) cudaEventDestroy(e);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
    b->push = nullptr;
    return LBG_OK;
}

lbg_status lbg_halo_push_connect(lbg_block b, const int (*offs)[3], const lbg_block* nbrs, int n) {
    if (lbg_status s_ = aa_refuse(b, "lbg_halo_push_connect")) return s_;
    if (!b || (n > 0 && (!offs || !nbrs))) return set_error(LBG_INVALID, "null argument");
    if (n > kMaxPush) return set_error(LBG_INVALID, "at most 26 halo neighbours");
    for (int t = 0; t < n; ++t) {
        if (!nbrs[t] || nbrs[t] == b) return set_error(LBG_INVALID, "push neighbours must be other blocks");
        bool face_or_edge = false;
        for (int d = 0; d < 3; ++d) {
            if (offs[t][d] < -1 || offs[t][d] > 1) return set_error(LBG_INVALID, "bad neighbour offset");
            face_or_edge = face_or_edge || offs[t][d] != 0;
        }
        if (!face_or_edge) return set_error(LBG_INVALID, "bad neighbour offset");
    }
    LBG_CUDA(cudaSetDevice(b->device));
    // peer access to every neighbour's device (stores into its buffers)
    for (int t = 0; t < n; ++t) {
        const int dev = nbrs[t]->device;
        if (dev == b->device) continue;
        int ok = 0;
        LBG_CUDA(cudaDeviceCanAccessPeer(&ok, b->device, dev));
        if (!ok) return set_error(LBG_CUDA_ERROR, "halo push: no peer access between the blocks' GPUs");
        const cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled)
            cudaGetLastError();
        else if (e != cudaSuccess)
            return cuda_check(e, "cudaDeviceEnablePeerAccess");
    }
    lbg_halo_push_destroy(b);
    auto* p = new Push;
    b->push = p;
    p->n = n;
    for (int t = 0; t < n; ++t) {
        for (int d = 0; d < 3; ++d) p->off[t][d] = offs[t][d];
        p->nbr[t] = nbrs[t];
    }
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    LBG_CUDA(cudaStreamCreateWithPriority(&p->stream, cudaStreamNonBlocking, hi_prio));
    LBG_CUDA(cudaEventCreateWithFlags(&p->ev_swept, cudaEventDisableTiming));
    for (auto& e : p->ev_push) LBG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return LBG_OK;
}

lbg_status lbg_halo_push(lbg_block b) {
    if (!b || !b->push) return set_error(LBG_INVALID, "lbg_halo_push_connect first");
    Push& p = *b->push;
    LBG_CUDA(cudaSetDevice(b->device));
    const long long step = p.count.load();
    PushArgs a{};
    a.err = b->err_d;
    a.n = 0;
    a.begin[0] = 0;
    const int nself[3] = {b->L.nx, b->L.ny, b->L.nz};
    for (int t = 0; t < p.n; ++t) {
        const int* o = p.off[t];
        lbg_block nb = p.nbr[t];
        const int nn[3] = {nb->L.nx, nb->L.ny, nb->L.nz};
        int nq = 0;
        for (int q = 0; q < kQ; ++q) {
            const int c[3] = {cx(q), cy(q), cz(q)};
            bool out = true;
            for (int d = 0; d < 3; ++d)
                if (o[d] != 0 && c[d] != o[d]) out = false;
            if (out) a.q[a.n][nq++] = q;
        }
        if (nq == 0) continue;  // corner: no D3Q19 velocity crosses it
        a.nq[a.n] = nq;
        long long cells = 1;
        for (int d = 0; d < 3; ++d) {
            // source_slab(o) (sim.cpp:120-135) and its place in the neighbour's ghost layer
            if (o[d] == 1) {
                a.lo[a.n][d] = nself[d] - 1;
                a.ext[a.n][d] = 1;
                a.sh[a.n][d] = -nself[d];  // n-1 -> -1
            } else if (o[d] == -1) {
                a.lo[a.n][d] = 0;
                a.ext[a.n][d] = 1;
                a.sh[a.n][d] = nn[d];  // 0 -> n_nbr
            } else {
                if (nn[d] != nself[d]) return set_error(LBG_INVALID, "halo push: neighbour face extents differ");
                a.lo[a.n][d] = 0;
                a.ext[a.n][d] = nself[d];
                a.sh[a.n][d] = b->lo[d] - nb->lo[d];
            }
            cells *= a.ext[a.n][d];
        }
        a.dst[a.n] = nb->buf[nb->cur ^ 1];
        a.px[a.n] = nb->L.px;
        a.py[a.n] = nb->L.py;
        a.plane[a.n] = nb->L.plane;
        a.begin[a.n + 1] = a.begin[a.n] + cells * nq;
        ++a.n;
    }
    // after this block's sweep (its dst is complete) ...
    LBG_CUDA(cudaEventRecord(p.ev_swept, b->stream));
    LBG_CUDA(cudaStreamWaitEvent(p.stream, p.ev_swept, 0));
    // ... and after each neighbour's previous sweep, the last reader of the buffer written here
    // (its push of step - 1 follows that sweep; every neighbour has issued it: lockstep phases)
    if (step > 0)
        for (int t = 0; t < p.n; ++t) {
            Push* q = p.nbr[t]->push;
            if (!q || q->count.load() < step) return set_error(LBG_SYNC_ERROR, "halo push: neighbour is behind");
            LBG_CUDA(cudaStreamWaitEvent(p.stream, q->ev_push[(step - 1) & 1], 0));
        }
    if (a.n > 0) {
        halo_push_kernel<<<(unsigned)((a.begin[a.n] + 255) / 256), 256, 0, p.stream>>>(b->dst(), b->L, a);
        LBG_LAUNCH_CHECK();
    }
    LBG_CUDA(cudaEventRecord(p.ev_push[step & 1], p.stream));
    p.count.store(step + 1);
    return LBG_OK;
}

lbg_status lbg_halo_push_wait(lbg_block b) {
    if (!b || !b->push) return set_error(LBG_INVALID, "lbg_halo_push_connect first");
    Push& p = *b->push;
    LBG_CUDA(cudaSetDevice(b->device));
    // the neighbours' pushes of the step this block last swept (its own count - 1): the same
    // step index on every block of a lockstep decomposition
    const long long want = p.count.load() - 1;
    if (want < 0) return set_error(LBG_SYNC_ERROR, "halo completion without a pending exchange");
    for (int t = 0; t < p.n; ++t) {
        Push* q = p.nbr[t]->push;
        if (!q || q->count.load() <= want) return set_error(LBG_SYNC_ERROR, "halo push of a neighbour is missing");
        LBG_CUDA(cudaStreamWaitEvent(b->stream, q->ev_push[want & 1], 0));
    }
    return LBG_OK;
}

}  // extern "C"
