// SPDX-License-Identifier: Apache-2.0
//
// lbg_run_host — Simulation::run(steps) (sim.cpp:702-704) of a periodic plain-fluid block whose
// PdfField lives in (pinned) host memory: upload, `steps` fused sweeps, download, with the three
// pipelined over z-slabs so both PCIe directions and the sweeps overlap. z is either wrapped
// in-kernel (one block spans the domain) or the slab axis of the NCCL halo (config 4: one block
// per GPU; the seam planes then take one halo exchange per step, see below).
//
// Schedule (one block, every axis wrapped in-kernel, double buffer A = buf[cur] / B):
//   * slab c (planes [cH, cH + H)) is copied H2D into a staging slot on `side` (19 linear copies,
//     one per q-plane run of the reference layout) and re-pitched into A on the compute stream;
//   * with planes [0, U) uploaded, step s can be computed on [s, U - s): its pulls need step s-1
//     on [s - 1, U - s + 1), and the planes below s wait for the z = 0 seam (their pulls wrap to
//     z = nz - 1). Each step s keeps a frontier F[s] and sweeps the new planes [F[s], U - s)
//     (src = step s-1's buffer, dst = step s's). A step s write to a plane p replaces step s-2's
//     value there, which step s-1 no longer needs: it has already swept up to F[s-1] = F[s] + 1;
//   * once the last slab is in, every step s (in order) sweeps the rest of the domain: [F[s], nz)
//     and the seam planes [0, s). With the NCCL halo on z, step s-1's planes 0 and nz-1 go to the
//     neighbours' z ghosts first (lbg_halo_begin/complete on step s-1's buffer; every rank makes
//     the same `steps` exchanges), which is the only time the planes next to the seam are pulled
//     from: the main phase never sweeps plane 0 or nz-1;
//   * the final step's planes go back to the host as soon as they are done: a pack kernel on its
//     own stream re-pitches them (interior cells from the final buffer, x/y ghost cells from A,
//     which holds the uploaded values — sweeps write interior cells only) into a staging slot,
//     and 19 D2H copies on a fourth stream write the slot's planes back into `host`.
// So the H2D copy engine, the D2H copy engine and the SMs work at the same time; the job's time
// is about one PCIe direction's transfer of the field plus the download of the last ~2 x steps
// planes (the seam cone), instead of the sum of both directions.
//
// The op sequence is lbg_job_schedule.hpp's (host-only; tests/test_job_schedule.py replays it
// against these double-buffer rules for 40,000 cases). The sweeps are K1 (sweep_planes ->
// sweep_box_kernel) on plane ranges: every interior cell gets
// exactly the operations of the whole-block sweep, so the result is bitwise that of
// upload + steps x (sweep + swap) + download (tests/test_gpu_job.py).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "lbg_internal.cuh"
#include "lbg_job_schedule.hpp"

namespace lbg {

constexpr int kJobSlots = 3;

// staging slot [q][zc][jj][ii] (zc < nzc, jj < py, ii < nx + 2: the reference layout's rows of
// planes z0 .. z0 + nzc - 1, ghost rows and columns included) -> device rows of `dev`
__global__ void __launch_bounds__(128) job_unpack_kernel(double* __restrict__ dev, const double* __restrict__ stg,
                                                          Layout L, int z0, int nzc) {
    const int w = L.nx + 2;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= w) return;
    const int jj = blockIdx.y;
    const int q = blockIdx.z / nzc, zc = blockIdx.z - q * nzc;
    const long long t = (((long long)q * nzc + zc) * L.py + jj) * w + c;
    const long long row = (long long)q * L.py * L.pz + (long long)(z0 + zc + 1) * L.py + jj;
    dev[row * L.px + (kXOff - 1) + c] = stg[t];
}

// the reverse for the download: interior cells from `fin`, the x/y ghost cells from `gh`
__global__ void __launch_bounds__(128) job_pack_kernel(const double* __restrict__ fin, const double* __restrict__ gh,
                                                        double* __restrict__ stg, Layout L, int z0, int nzc) {
    const int w = L.nx + 2;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= w) return;
    const int jj = blockIdx.y;
    const int q = blockIdx.z / nzc, zc = blockIdx.z - q * nzc;
    const long long t = (((long long)q * nzc + zc) * L.py + jj) * w + c;
    const long long row = (long long)q * L.py * L.pz + (long long)(z0 + zc + 1) * L.py + jj;
    const long long off = row * L.px + (kXOff - 1) + c;
    const bool interior = c >= 1 && c <= L.nx && jj >= 1 && jj <= L.ny;
    stg[t] = interior ? fin[off] : gh[off];
}

void free_job(lbg_block b) {
    for (int s = 0; s < kJobSlots; ++s) {
        if (b->job_up[s]) cudaFree(b->job_up[s]);
        if (b->job_dn[s]) cudaFree(b->job_dn[s]);
        b->job_up[s] = b->job_dn[s] = nullptr;
        for (int e = 0; e < 4; ++e)
            if (b->job_ev[e][s]) {
                cudaEventDestroy(b->job_ev[e][s]);
                b->job_ev[e][s] = nullptr;
            }
    }
    b->job_cap = 0;
    if (b->job_pack) cudaStreamDestroy(b->job_pack);
    if (b->job_d2h) cudaStreamDestroy(b->job_d2h);
    b->job_pack = b->job_d2h = nullptr;
}

static lbg_status ensure_job(lbg_block b, size_t cap) {
    if (b->job_cap < cap) {
        for (int s = 0; s < kJobSlots; ++s) {
            if (b->job_up[s]) cudaFree(b->job_up[s]);
            if (b->job_dn[s]) cudaFree(b->job_dn[s]);
            b->job_up[s] = b->job_dn[s] = nullptr;
        }
        b->job_cap = 0;
        for (int s = 0; s < kJobSlots; ++s) {
            LBG_CUDA(cudaMalloc(&b->job_up[s], sizeof(double) * cap));
            LBG_CUDA(cudaMalloc(&b->job_dn[s], sizeof(double) * cap));
        }
        b->job_cap = cap;
    }
    if (!b->job_pack) LBG_CUDA(cudaStreamCreateWithFlags(&b->job_pack, cudaStreamNonBlocking));
    if (!b->job_d2h) LBG_CUDA(cudaStreamCreateWithFlags(&b->job_d2h, cudaStreamNonBlocking));
    for (int e = 0; e < 4; ++e)
        for (int s = 0; s < kJobSlots; ++s)
            if (!b->job_ev[e][s]) LBG_CUDA(cudaEventCreateWithFlags(&b->job_ev[e][s], cudaEventDisableTiming));
    return LBG_OK;
}

}  // namespace lbg

using namespace lbg;

extern "C" lbg_status lbg_run_host(lbg_block b, const lbg_fluid* fl, double* host, int steps, int slab_planes,
                                   lbg_errors* out) {
    if (!b || !fl || !host) return set_error(LBG_INVALID, "null argument");
    if (!(fl->tau > 0.5))  // FluidParams::validate (lbm.hpp:28-32)
        return set_error(LBG_CONFIG_ERROR, "fluid relaxation time tau must be > 0.5 (got " + std::to_string(fl->tau) + ")");
    if (steps < 0) return set_error(LBG_INVALID, "negative step count");
    if (b->coupling) return set_error(LBG_INVALID, "lbg_run_host: plain-fluid blocks only");
    if (b->aa) return set_error(LBG_INVALID, "lbg_run_host: not available on an AA-streaming block");
    // z: wrapped in-kernel (the whole periodic domain), or the slab axis of an NCCL halo
    // (lbg_comm_init; its exchanges run at the seam, once per step, in the tail)
    const bool zcomm = !b->wrap[2] && comm_axis(b) == 2;
    if (!(b->wrap[0] && b->wrap[1] && (b->wrap[2] || zcomm)))
        return set_error(LBG_INVALID, "lbg_run_host: x and y must be periodic and wrapped in-kernel, z wrapped or "
                                      "the slab axis of the block's NCCL halo");
    const Layout& L = b->L;
    const int nz = L.nz;
    const int H = std::max(1, std::min({slab_planes > 0 ? slab_planes : 16, nz, 2048}));  // grid.z = 19 H
    const int w = L.nx + 2;
    const size_t run = (size_t)L.py * w;  // doubles of one reference-layout z-plane of one q
    LBG_CUDA(cudaSetDevice(b->device));
    if (lbg_status s = ensure_job(b, (size_t)kQ * H * run)) return s;
    cudaStream_t up = b->side, cs = b->stream, pk = b->job_pack, dl = b->job_d2h;
    // one event per recorded point that another stream waits on once (download pieces)
    std::vector<cudaEvent_t> evs;
    auto fresh_event = [&](cudaEvent_t& ev) -> lbg_status {
        LBG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        evs.push_back(ev);
        return LBG_OK;
    };
    // everything queued on the block's streams before the job comes first
    cudaEvent_t ev_start;
    if (lbg_status s = fresh_event(ev_start)) return s;
    LBG_CUDA(cudaEventRecord(ev_start, cs));
    LBG_CUDA(cudaStreamWaitEvent(up, ev_start, 0));
    LBG_CUDA(cudaStreamWaitEvent(pk, ev_start, 0));
    LBG_CUDA(cudaStreamWaitEvent(dl, ev_start, 0));

    double* A = b->buf[b->cur];
    double* B = b->buf[b->cur ^ 1];
    double* fin = (steps & 1) ? B : A;
    auto src_of = [&](int s) { return ((s - 1) & 1) ? B : A; };
    auto dst_of = [&](int s) { return (s & 1) ? B : A; };
    const unsigned gx = (unsigned)((w + 127) / 128);

    int dn_piece = 0, up_chunk = 0;
    // one download piece (<= H planes of the final step, done on the compute stream so far)
    auto download = [&](int a, int nzc) -> lbg_status {
        const int slot = dn_piece % kJobSlots;
        cudaEvent_t ev;  // the final step is done on [a, a + nzc)
        if (lbg_status s = fresh_event(ev)) return s;
        LBG_CUDA(cudaEventRecord(ev, cs));
        LBG_CUDA(cudaStreamWaitEvent(pk, ev, 0));
        if (dn_piece >= kJobSlots) LBG_CUDA(cudaStreamWaitEvent(pk, b->job_ev[3][slot], 0));
        job_pack_kernel<<<dim3(gx, (unsigned)L.py, (unsigned)(kQ * nzc)), 128, 0, pk>>>(fin, A, b->job_dn[slot], L, a,
                                                                                      nzc);
        LBG_LAUNCH_CHECK();
        LBG_CUDA(cudaEventRecord(b->job_ev[2][slot], pk));
        LBG_CUDA(cudaStreamWaitEvent(dl, b->job_ev[2][slot], 0));
        for (int q = 0; q < kQ; ++q)
            LBG_CUDA(cudaMemcpyAsync(host + ((size_t)q * L.pz + a + 1) * run, b->job_dn[slot] + (size_t)q * nzc * run,
                                     sizeof(double) * nzc * run, cudaMemcpyDeviceToHost, dl));
        LBG_CUDA(cudaEventRecord(b->job_ev[3][slot], dl));
        ++dn_piece;
        return LBG_OK;
    };
    // one upload slab: H2D into a staging slot on `side`, re-pitched into A on the compute stream
    auto upload = [&](int z0, int nzc) -> lbg_status {
        const int slot = up_chunk % kJobSlots;
        if (up_chunk >= kJobSlots) LBG_CUDA(cudaStreamWaitEvent(up, b->job_ev[1][slot], 0));  // slot unpacked
        for (int q = 0; q < kQ; ++q)
            LBG_CUDA(cudaMemcpyAsync(b->job_up[slot] + (size_t)q * nzc * run, host + ((size_t)q * L.pz + z0 + 1) * run,
                                     sizeof(double) * nzc * run, cudaMemcpyHostToDevice, up));
        LBG_CUDA(cudaEventRecord(b->job_ev[0][slot], up));
        LBG_CUDA(cudaStreamWaitEvent(cs, b->job_ev[0][slot], 0));
        job_unpack_kernel<<<dim3(gx, (unsigned)L.py, (unsigned)(kQ * nzc)), 128, 0, cs>>>(A, b->job_up[slot], L, z0, nzc);
        LBG_LAUNCH_CHECK();
        LBG_CUDA(cudaEventRecord(b->job_ev[1][slot], cs));
        ++up_chunk;
        return LBG_OK;
    };
    // step s-1's planes 0 and nz-1 into the neighbours' z ghosts (NCCL halo on step s-1's buffer)
    auto seam = [&](int s) -> lbg_status {
        const int cur0 = b->cur;
        b->cur = (src_of(s) == b->buf[0]) ? 0 : 1;
        lbg_status st = lbg_halo_begin(b);
        if (st == LBG_OK) st = lbg_halo_complete(b);
        b->cur = cur0;
        return st;
    };

    // the whole schedule (lbg_job_schedule.hpp) is enqueued by `schedule`; whatever it returns,
    // every stream of the job is drained below before the host buffer is handed back (no copy
    // may still target it)
    auto schedule = [&]() -> lbg_status {
        // LBG_JOB_TAIL=k: the last slab uploaded in pieces of H / k planes (A/B; default 0, whole
        // slabs: measured no faster at 512^3, 20 steps — profiles/r02_ab_job.txt)
        static const int tail = [] {
            const char* e = std::getenv("LBG_JOB_TAIL");
            return e ? std::atoi(e) : 0;
        }();
        for (const job::Item& it : job::schedule(nz, steps, H, zcomm, tail)) {
            lbg_status st = LBG_OK;
            switch (it.op) {
                case job::Op::Upload: st = upload(it.z0, it.z1 - it.z0); break;
                case job::Op::Sweep: st = sweep_planes(b, fl, src_of(it.s), dst_of(it.s), it.z0, it.z1, cs); break;
                case job::Op::Seam: st = seam(it.s); break;
                case job::Op::Download: st = download(it.z0, it.z1 - it.z0); break;
            }
            if (st != LBG_OK) return st;
        }
        return LBG_OK;
    };
    const lbg_status st = schedule();
    // drain every stream of the job before touching the host buffer or the block again
    cudaError_t e1 = cudaStreamSynchronize(dl), e2 = cudaStreamSynchronize(pk), e3 = cudaStreamSynchronize(up),
                e4 = cudaStreamSynchronize(cs);
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);
    if (st != LBG_OK) return st;
    for (cudaError_t e : {e1, e2, e3, e4})
        if (e != cudaSuccess) return set_error(LBG_CUDA_ERROR, std::string("lbg_run_host: ") + cudaGetErrorString(e));
    b->cur ^= (steps & 1);
    return lbg_sync(b, out);  // the accumulated end-of-sweep checks (NumericError)
}
