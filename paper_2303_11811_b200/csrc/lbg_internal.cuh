// SPDX-License-Identifier: Apache-2.0
//
// Private types of liblbg: the device block, its HBM layout and the D3Q19 tables.
//
// HBM layout of one PDF buffer (the reference's PdfField, field.hpp:36-78, re-laid out
// for sm_100a coalescing):
//   19 q-planes back to back, plane stride = px * py * pz doubles (py = ny+2, pz = nz+2),
//   row (j,k) at ((k+1)*py + (j+1)) * px, cell i at row + kXOff + i.
//   kXOff = 16 puts interior i = 0 on a 128-byte boundary; px is a multiple of 16, so
//   every interior row starts line-aligned and a warp's 32 consecutive cells are exactly
//   two 128-B lines per q-plane. The x ghost (i = -1) sits at kXOff - 1.
// Coupling fields keep the reference's interior lexicographic layout (field.hpp:95-97).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "lbg.h"

namespace lbg {

constexpr int kQ = 19;
constexpr int kXOff = 16;

// lattice.hpp:18-29 (rest, then opposite pairs) and 32-39 (weights over 36).
__host__ __device__ constexpr int cx(int q) {
    constexpr int t[kQ] = {0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0};
    return t[q];
}
__host__ __device__ constexpr int cy(int q) {
    constexpr int t[kQ] = {0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1};
    return t[q];
}
__host__ __device__ constexpr int cz(int q) {
    constexpr int t[kQ] = {0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1};
    return t[q];
}
__host__ __device__ constexpr int wnum(int q) {
    constexpr int t[kQ] = {12, 2, 2, 2, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    return t[q];
}
// kW[q] = kWeightNum36[q] / 36.0, rounded once exactly like lattice.hpp:35-39.
__host__ __device__ constexpr double wq(int q) { return wnum(q) / 36.0; }
__host__ __device__ constexpr int opposite(int q) { return q == 0 ? 0 : (((q - 1) ^ 1) + 1); }

constexpr double kMaxVelocity = 0.57;  // lbm.hpp:19

struct Layout {
    int nx, ny, nz;
    int px, py, pz;
    long long plane;  // doubles per q-plane
    __host__ __device__ long long row(int j, int k) const {
        return ((long long)(k + 1) * py + (j + 1)) * px + kXOff;
    }
    __host__ __device__ long long idx(int i, int j, int k) const { return row(j, k) + i; }
    __host__ __device__ long long shift(int q) const {
        return cx(q) + (long long)cy(q) * px + (long long)cz(q) * px * py;
    }
    __host__ __device__ long long frac(int i, int j, int k) const {
        return ((long long)k * ny + j) * nx + i;
    }
};

struct DeviceErrors {
    unsigned long long unstable;
    unsigned long long overfull;
    unsigned long long unknown;
    unsigned long long p2p_timeout;  // lbg_p2p.cu wait gave up
    unsigned long long oob;          // checked build: an index outside its buffer (access skipped)
    unsigned long long race;         // checked build: a cell written != once by one sweep
};

// Checked build (make checked, -DLBG_CHECKED): the hot kernels check every computed index
// against its buffer (an out-of-range one is counted and redirected to element 0, so the run
// goes on and lbg_sync reports it) and every sweep counts the cells it writes (each cell of
// the swept box exactly once across all the kernels of the sweep: K12 || two-entry K2, K1 ||
// K2, ... — a double write is a race between them, a missing one a hole). compute-sanitizer is
// closed on the GPU pool; this is the repository's own memcheck/racecheck substitute.
#ifdef LBG_CHECKED
#define LBG_IDX(idx, limit, err) ::lbg::checked_idx((long long)(idx), (long long)(limit), (err))
#else
#define LBG_IDX(idx, limit, err) (idx)
#endif
__device__ __forceinline__ long long checked_idx(long long idx, long long limit, DeviceErrors* err) {
    if (idx < 0 || idx >= limit) {
        atomicAdd(&err->oob, 1ull);
        return 0;
    }
    return idx;
}

struct TimedSpan {
    int cat;
    cudaEvent_t a, b;
};

// snapshot_index (psm.cpp:46-51): id -> index in the id-sorted snapshot list. A dense table
// over [id_min, id_min + range) is built at every snapshot upload when the ids are dense
// enough (the usual case: particle ids 0..N-1); otherwise a binary search. Either way an
// absent id gives -1.
struct SnapIndex {
    const lbg_snapshot* s;
    int n;
    const int* tab;  // nullptr: binary search
    int id_min;
    int range;
    __device__ __forceinline__ int operator()(int id) const {
        if (tab) {
            const long long o = (long long)id - id_min;
            return (o >= 0 && o < range) ? tab[o] : -1;
        }
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s[mid].id < id)
                lo = mid + 1;
            else
                hi = mid;
        }
        return (lo < n && s[lo].id == id) ? lo : -1;
    }
};

// The state one mapping produces (the fraction field, its segment lists, the snapshot list it
// was mapped from with its index, and the host bookkeeping about that list). lbg_map_prepare
// maps into a shadow copy while the block keeps using (and observers keep seeing) the current
// one; lbg_map_commit swaps the two by pointer.
struct MapState {
    uint8_t* count = nullptr;
    int* id0 = nullptr;
    int* id1 = nullptr;
    int* pidx0 = nullptr;
    double* b0 = nullptr;
    double* b1 = nullptr;
    double* btot = nullptr;
    unsigned* seg_list = nullptr;
    // covered-segment counts of the last mapping, copied to the host asynchronously (the
    // coupled sweep picks the unified kernel or the split by the covered fraction)
    int* segn_h = nullptr;
    cudaEvent_t ev_segn = nullptr;
    bool segn_pending = false;
    int* seg_n = nullptr;
    lbg_snapshot* snaps_d = nullptr;
    int snaps_dcap = 0;
    int n_snaps = 0;
    int* snap_tab = nullptr;
    long long snap_tab_cap = 0;
    int snap_id_min = 0;
    int snap_range = 0;
    std::vector<int> map_ids;
    std::vector<lbg_snapshot> map_snaps;
    bool map_ids_valid = false;
    bool v_snap = false;
    bool p_direct = false;
    bool cov_dirty = true;
};

struct Comm;  // lbg_halo.cu
struct P2P;   // lbg_p2p.cu
struct Push;  // lbg_push.cu

struct MapRec;  // lbg_psm.cu

}  // namespace lbg

struct lbg_block_s {
    int device = 0;
    int lo[3] = {0, 0, 0};
    bool coupling = false;
    lbg::Layout L{};
    double* buf[2] = {nullptr, nullptr};
    int cur = 0;  // src = buf[cur], dst = buf[cur ^ 1]

    // coupling fields (interior lexicographic)
    uint8_t* count = nullptr;
    int* id0 = nullptr;
    int* id1 = nullptr;
    double* b0 = nullptr;
    double* b1 = nullptr;
    double* btot = nullptr;
    double* v0 = nullptr;  // xyz per cell
    double* v1 = nullptr;
    // v_snap: the solid velocities are those set_solid_velocities would compute from the
    // current snapshots over the current fraction field; the PSM kernels evaluate
    // u + omega x (c - x) inline instead of reading v0/v1 (which are then stale until
    // materialised by setu_kernel on download or before a fraction upload)
    bool v_snap = false;
    // pidx0: entry 0's index in the mapping list, written by the mapping kernel; valid for the
    // sweep while the current list is the mapping list (same ids in the same order)
    int* pidx0 = nullptr;
    bool p_direct = false;
    // ids of the snapshot list the fraction field was mapped from (valid after lbg_map):
    // a later set_solid_velocities list holding all of them cannot meet an unknown id
    std::vector<int> map_ids;
    bool map_ids_valid = false;
    double* m0 = nullptr;
    double* m1 = nullptr;
    // segment lists stale (after a fraction upload): rebuilt before the next sweep
    bool cov_dirty = true;
    // aligned 32-cell row segments holding covered cells (first cell index): segments with
    // one-entry cells only from the front (seg_n[0]), with a two-entry cell from the back
    unsigned* seg_list = nullptr;
    // covered-segment counts of the last mapping, copied to the host asynchronously (the
    // coupled sweep picks the unified kernel or the split by the covered fraction)
    int* segn_h = nullptr;
    cudaEvent_t ev_segn = nullptr;
    bool segn_pending = false;
    int* seg_n = nullptr;
    long long seg_cap = 0;

    // periodic axes the sweep wraps in-kernel (no ghost read), lbg_set_periodic_wrap
    int wrap[3] = {0, 0, 0};

    // force mode: LBG_FORCE_SCRATCH (reference: per-cell m scratch + finalize walk) or
    // LBG_FORCE_FUSED (the PSM kernel accumulates per-particle force/torque with warp
    // aggregation + atomics; the scratch is never written)
    int force_mode = 0;
    double* facc = nullptr;  // n_snaps x 6 (f xyz, t xyz)
    int* fused_used = nullptr;
    int facc_cap = 0;

    // particle snapshots: pinned staging + device copy (H2D on the side stream)
    lbg_snapshot* snaps_h = nullptr;
    lbg_snapshot* snaps_d = nullptr;
    int snaps_cap = 0;   // pinned staging
    int snaps_dcap = 0;  // device list
    int n_snaps = 0;
    int* snap_tab = nullptr;  // dense id -> index table (SnapIndex)
    long long snap_tab_cap = 0;
    int snap_id_min = 0;
    int snap_range = 0;  // 0: no table (sparse ids)
    lbg::MapState* shadow = nullptr;  // lbg_map_prepare's target
    bool prepared = false;
    bool preparing = false;
    // device binning for the mapping kernel (lbg_psm.cu)
    int* bin_count = nullptr;
    int* bin_start = nullptr;
    int* bin_items = nullptr;
    long long bin_items_cap = 0;
    lbg::MapRec* bin_rec = nullptr;  // the items' candidate records (sorted like the items)
    long long bin_rec_cap = 0;
    long long n_bins_cap = 0;
    // hydro reduction scratch
    double* red_rows = nullptr;  // n_snaps x 12
    int* red_used = nullptr;
    int red_cap = 0;
    double* red_rows_h = nullptr;
    int* red_used_h = nullptr;
    // box-walk reduction: per-particle cell boxes (generic source), the mapping list's
    // snapshots (the reach boxes are valid while the list keeps their positions and radii)
    int* red_box = nullptr;
    int red_box_cap = 0;
    std::vector<lbg_snapshot> map_snaps;
    cudaEvent_t ev_red = nullptr;

    lbg::DeviceErrors* err_d = nullptr;
    int* wcount = nullptr;  // checked build: per-cell write counts of the current sweep
    lbg::DeviceErrors* err_h = nullptr;  // pinned

    cudaStream_t stream = nullptr;  // compute
    cudaStream_t side = nullptr;    // H2D/D2H of particle data
    cudaEvent_t ev_side = nullptr;
    // coupled sweeps: K2 (covered segments) runs on `aux` concurrently with K1 on `stream`
    // (disjoint cells); fork/join by events
    cudaStream_t aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    bool timing = false;
    std::vector<lbg::TimedSpan> spans;
    std::vector<cudaEvent_t> event_pool;
    double acc_ms[LBG_NUM_CATS] = {};
    long long acc_n[LBG_NUM_CATS] = {};

    lbg::Comm* comm = nullptr;
    lbg::P2P* p2p = nullptr;
    lbg::Push* push = nullptr;
    long long device_bytes = 0;
    double* obs_d = nullptr;  // observer partials (lbg_observe)
    double* obs_h = nullptr;
    double* mom_d = nullptr;  // per-cell moments staging (lbg_moments)
    size_t mom_cap = 0;

    // device-side generic halo (lbg_halo_stage / lbg_halo_fetch): staged source slabs per
    // neighbour offset (index (ox+1)*9+(oy+1)*3+(oz+1)), a receive buffer, a staging event
    double* stage[27] = {};
    size_t stage_cap[27] = {};
    double* recv_buf = nullptr;
    size_t recv_cap = 0;
    double* recv_multi[27] = {};  // lbg_halo_fetch_all: per-direction receive slots (peer copies)
    size_t recv_multi_cap[27] = {};
    cudaEvent_t ev_stage = nullptr;
    // staging reuse: fetches that read this block's staging record their stream's event here
    // (under the mutex: receivers run on their own worker threads); the next lbg_halo_stage
    // waits on them before overwriting the staging buffers
    std::mutex consumers_mu;
    std::vector<cudaEvent_t> consumers;
    cudaEvent_t ev_fetched = nullptr;  // recorded after this block's fetch/unpack

    // pinned-host PDF transfers: double-buffered device staging (lbg_core.cu)
    double* xfer[2] = {nullptr, nullptr};
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};

    // streamed host job (lbg_run_host, lbg_job.cu): z-slab staging slots per direction (doubles
    // per slot: job_cap), the pack and D2H streams, per-slot events (0 uploaded, 1 unpacked,
    // 2 packed, 3 downloaded)
    double* job_up[3] = {nullptr, nullptr, nullptr};
    double* job_dn[3] = {nullptr, nullptr, nullptr};
    size_t job_cap = 0;
    cudaStream_t job_pack = nullptr, job_d2h = nullptr;
    cudaEvent_t job_ev[4][3] = {};

    // AA in-place streaming (lbg_aa.cu): one buffer (buf[cur]); aa_phase 0: state S0 (the
    // double-buffer src), 1: S1 (streamed, slots swapped); aa_pending: swept, not yet swapped
    bool aa = false;
    int aa_phase = 0;
    bool aa_pending = false;

    double* src() const { return buf[cur]; }
    double* dst() const { return buf[cur ^ 1]; }
};

namespace lbg {

// AA streaming (lbg_aa.cu): one step of the in-place sweep; the S0 image of an S1 buffer
lbg_status aa_sweep(lbg_block b, const lbg_fluid* fl);
lbg_status aa_unstream(lbg_block b, double* out);
// K1 over z-planes [z0, z1) from src into dst on stream st (lbg_sweep.cu; the host job's sweeps)
lbg_status sweep_planes(lbg_block b, const lbg_fluid* fl, const double* src, double* dst, int z0, int z1,
                        cudaStream_t st);
// the slab axis of the block's NCCL halo (lbg_comm_init), -1 if none (lbg_halo.cu)
int comm_axis(lbg_block b);
// releases the host job's staging, streams and events (lbg_job.cu)
void free_job(lbg_block b);
// frees the shadow mapping state of lbg_map_prepare (lbg_psm.cu)
void free_shadow(lbg_block b);
// covered-cell counts and segment lists rebuilt from `count` (lbg_psm.cu)
lbg_status rebuild_covered(lbg_block b);
// the covered-segment counts to the host, asynchronously (lbg_psm.cu)
lbg_status post_segment_counts(lbg_block b);
// the block's current snapshot index
inline SnapIndex snap_index(const lbg_block_s* b) {
    return SnapIndex{b->snaps_d, b->n_snaps, b->snap_range > 0 ? b->snap_tab : nullptr, b->snap_id_min,
                     b->snap_range};
}

// warp-aggregated append of `pred` lanes' values to list[*n ...]
__device__ __forceinline__ void warp_append(bool pred, unsigned v, unsigned* list, int* n) {
    const unsigned m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(n, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane) - 1))] = v;
}

// error plumbing (lbg_core.cu)
lbg_status set_error(lbg_status s, const std::string& msg);
lbg_status cuda_check(cudaError_t e, const char* what);
void count_launch();
// operations defined on the double-buffered layout refuse an AA block (`state1`: only while it
// holds the streamed state S1)
inline lbg_status aa_refuse(lbg_block b, const char* what, bool state1 = false) {
    if (b && b->aa && (!state1 || b->aa_phase == 1))
        return set_error(LBG_INVALID, std::string(what) + ": not available on an AA-streaming block" +
                                          (state1 ? " after an odd number of steps" : ""));
    return LBG_OK;
}

// Grow-only device buffer: holds at least `need` elements afterwards (`want` when it has to
// grow, for geometric growth). The old buffer is freed first; on failure the pointer is null
// and the capacity 0, so no later call sees a stale capacity over a freed buffer. Callers
// order the free after pending work (the buffers are per block and used on its streams).
template <class T, class C>
inline lbg_status grow_device(T*& p, C& cap, long long need, long long want, const char* what) {
    if (p && (long long)cap >= need) return LBG_OK;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const long long n = need > want ? need : want;
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, sizeof(T) * (size_t)n);
    if (e != cudaSuccess) return cuda_check(e, what);
    p = static_cast<T*>(q);
    cap = static_cast<C>(n);
    return LBG_OK;
}

// timing spans around a launch (no-ops unless timing is on)
struct Span {
    lbg_block b;
    int cat;
    cudaEvent_t a = nullptr;
    Span(lbg_block b_, int cat_);
    ~Span();
};

}  // namespace lbg

#define LBG_CUDA(call)                                                      \
    do {                                                                    \
        cudaError_t e_ = (call);                                            \
        if (e_ != cudaSuccess) return ::lbg::cuda_check(e_, #call);         \
    } while (0)

#define LBG_LAUNCH_CHECK()                                                  \
    do {                                                                    \
        ::lbg::count_launch();                                              \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) return ::lbg::cuda_check(e_, "kernel launch"); \
    } while (0)
