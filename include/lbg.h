/* SPDX-License-Identifier: Apache-2.0
 *
 * lbg.h — C-ABI of the B200-native GPU side of the arXiv 2303.11811 coupled
 * LBM/PSM/DEM solver. Plain pointers and sizes, no C++ or torch types, never throws.
 *
 * Every entry point replaces one operator of the reference C++ library
 * (/root/reference/proj, "lbdem"); the citation next to each declaration names the
 * reference interface it stands in for. A block (lbg_block) is the device-side twin of
 * the reference's BlockState fields (sim.hpp:28-52): the double-buffered PdfField, and
 * with `coupling` the FractionField, SolidVelocityField and CellMomentumScratch.
 *
 * Layout contract for host buffers (so parity tests compare raw arrays):
 *   PDF:       19 q-planes of (nx+2)(ny+2)(nz+2) doubles, PdfField::idx order
 *              ((k+1)(ny+2)+(j+1))(nx+2)+(i+1)                   (field.hpp:47-49)
 *   fraction:  interior cells, (k*ny+j)*nx+i                       (field.hpp:95-97)
 *   Vec3 data: xyz interleaved per cell                            (field.hpp:101-118)
 * The device layout is private (x-pitch padded for 128-byte row alignment).
 *
 * Asynchrony: calls enqueue work on the block's CUDA streams and return. Errors the
 * reference raises at the end of an operator (NumericError for unstable cells or
 * overfull cells, SyncError for unknown particle ids) are accumulated in device
 * counters and reported by lbg_sync(), which maps them to LBG_NUMERIC_ERROR /
 * LBG_SYNC_ERROR with the reference's messages (lbm.cpp:47-48, psm.cpp:133-135,
 * psm.cpp:167-168, psm.cpp:301-303). Threading: a block belongs to one host thread at a
 * time, like a BlockState.
 */
#ifndef LBG_H
#define LBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; 1-4 map to the reference exceptions (errors.hpp:10-32, CLI exit codes
 * lbdem_cli.cpp:199-214). */
typedef enum {
    LBG_OK = 0,
    LBG_CONFIG_ERROR = 1,  /* ConfigError  */
    LBG_NUMERIC_ERROR = 2, /* NumericError */
    LBG_SYNC_ERROR = 3,    /* SyncError    */
    LBG_IO_ERROR = 4,      /* IoError      */
    LBG_CUDA_ERROR = 5,    /* CUDA/NCCL runtime failure (no reference twin) */
    LBG_INVALID = 6        /* bad argument / missing coupling fields */
} lbg_status;

typedef struct lbg_block_s* lbg_block;

/* CellBox (field.hpp:13-30): half-open [lo, hi) in block-local cell coordinates. */
typedef struct {
    int lo[3];
    int hi[3];
} lbg_box;

/* FluidParams (lbm.hpp:21-33). */
typedef struct {
    double tau;
    double f_ext[3];
} lbg_fluid;

/* BcKind / FaceBc (boundary.hpp:11-17). Face order -x,+x,-y,+y,-z,+z (boundary.hpp:20). */
enum { LBG_BC_PERIODIC = 0, LBG_BC_NO_SLIP = 1, LBG_BC_VELOCITY = 2, LBG_BC_PRESSURE = 3 };
typedef struct {
    int kind;
    int pad_;
    double u_wall[3];
    double rho;
} lbg_face_bc;

/* ParticleSnapshot (psm.hpp:16-23), id-sorted list of locals + ghosts. */
typedef struct {
    int id;
    int pad_;
    double x[3];
    double r;
    double f_r;
    double u[3];
    double omega[3];
} lbg_snapshot;

/* HydroPartial (psm.hpp:88-92): Neumaier (sum, comp) pairs, vec3.hpp:71-95. */
typedef struct {
    int id;
    int pad_;
    double f[3];
    double f_comp[3];
    double t[3];
    double t_comp[3];
} lbg_hydro_partial;

/* End-of-operator error counters (the reference's `bad`, `overfull`, `unknown`). */
typedef struct {
    long long unstable_cells; /* lbm.cpp:33-48, psm.cpp:233-261 */
    long long overfull_cells; /* psm.cpp:132-135 */
    long long unknown_ids;    /* psm.cpp:166-168, 300-303 */
} lbg_errors;

/* Hydrodynamic reduction modes for lbg_reduce_hydro. */
enum {
    LBG_REDUCE_PARITY = 0, /* per-particle lexicographic Neumaier walk: bitwise == reference */
    LBG_REDUCE_FAST = 1    /* warp shuffles + shared memory + per-particle atomics (tolerance) */
};

/* Where the PSM kernel puts the per-entry momentum transfer. */
enum {
    LBG_FORCE_SCRATCH = 0, /* CellMomentumScratch m0/m1 (field.hpp:112-118), reduced by
                              lbg_reduce_hydro; PARITY-capable (reference semantics) */
    LBG_FORCE_FUSED = 1    /* summed per particle inside the sweep (warp-aggregated by particle,
                              one atomic per warp group); lbg_reduce_hydro(FAST) returns the sums */
};

/* Timing categories, perf.hpp:17-26 (perf::Category order). */
enum {
    LBG_CAT_PSM = 0,
    LBG_CAT_PSM_COMM = 1,
    LBG_CAT_MAPPING = 2,
    LBG_CAT_SETU = 3,
    LBG_CAT_REDF = 4,
    LBG_CAT_PD = 5,
    LBG_CAT_PD_COMM = 6,
    LBG_CAT_OTHER = 7,
    LBG_NUM_CATS = 8
};

/* ------------------------------------------------------------------ library */
const char* lbg_last_error(void);           /* message of the last failing call (thread-local) */
const char* lbg_version(void);
int lbg_device_count(void);

/* Pinned host memory for async H2D/D2H (the "pinned async copies" of the north star). */
lbg_status lbg_host_alloc(size_t bytes, void** out);
lbg_status lbg_host_free(void* p);

/* ------------------------------------------------------------------ block lifecycle */
/* BlockState ctor (sim.cpp:15-25) + PdfField(nx,ny,nz) (field.cpp:6-13): zeroed buffers. */
lbg_status lbg_block_create(int device, const int box_lo[3], const int dims[3], int coupling,
                            lbg_block* out);
lbg_status lbg_block_destroy(lbg_block b);
lbg_status lbg_block_info(lbg_block b, int dims[3], int box_lo[3], int* coupling,
                          long long* device_bytes);
/* cudaStream_t of the compute stream, for callers that time with their own events. */
void* lbg_block_stream(lbg_block b);

/* ------------------------------------------------------------------ PdfField access */
/* PdfField::src()/at_src() (field.hpp:56-62): whole src/dst buffer incl. ghosts. */
lbg_status lbg_upload_src(lbg_block b, const double* host);
lbg_status lbg_download_src(lbg_block b, double* host);
lbg_status lbg_upload_dst(lbg_block b, const double* host);
lbg_status lbg_download_dst(lbg_block b, double* host);
/* Simulation::initialize_fluid (sim.cpp:54-57) via PdfField::fill_src (field.cpp:15-22). */
lbg_status lbg_fill_equilibrium(lbg_block b, double rho, const double u[3]);
/* Shear-wave equilibrium state of validation.cpp:46-63 over a global `domain`, computed on
 * the device (synthetic benchmark input for configs 2/4; not bitwise with glibc sin/cos). */
lbg_status lbg_init_shear_wave(lbg_block b, const int domain[3]);
/* PdfField::fill_ghosts_src (field.cpp:24-35), NaN-poisoning tests. */
lbg_status lbg_fill_ghosts_src(lbg_block b, double v);
/* PdfField::swap (field.hpp:64). */
lbg_status lbg_swap(lbg_block b);
/* Simulation::run(steps) (sim.cpp:702-704) of a periodic plain-fluid block — x and y wrapped
 * in-kernel, z wrapped too (one block spans the domain) or the slab axis of the block's NCCL
 * halo (lbg_comm_init, axis 2; one block per rank, every rank calls this with the same
 * `steps`) — for a caller whose PdfField lives on the host: `host` (reference layout incl. ghosts, as lbg_upload_src) is the state before the
 * first step and receives, in place, the state after `steps` collide-stream steps. The
 * upload, the sweeps and the download are pipelined over z-slabs of `slab_planes` planes (0:
 * 16): slabs are uploaded in z order, step s of a plane range runs as soon as step s-1 of its
 * neighbour planes is done (the ranges next to the z = 0 seam last; with the NCCL halo the seam
 * planes take one halo exchange per step), and a slab goes back to
 * the host as soon as its last step is done, so H2D, D2H (separate streams, both PCIe
 * directions) and the sweeps overlap. Interior cells are bitwise those of lbg_upload_src +
 * steps x (lbg_sweep of the block + lbg_swap) + lbg_download_src; ghost cells keep their input
 * values. Afterwards the block's src holds the final state. The end-of-sweep stability checks
 * are accumulated and reported once, as lbg_sync does (LBG_NUMERIC_ERROR; `out` optional).
 * `host` should be pinned (lbg_host_alloc) for the copies to overlap. */
lbg_status lbg_run_host(lbg_block b, const lbg_fluid* fluid, double* host, int steps, int slab_planes,
                        lbg_errors* out);

/* ------------------------------------------------------------------ fluid operators */
/* collide_stream_* / psm_collide_stream_* over a CellBox (lbm.cpp:21-59, psm.cpp:218-276).
 * The plain or coupled kernel is chosen by the block's `coupling` flag, as
 * Simulation::run_kernel does (sim.cpp:221-236). */
lbg_status lbg_sweep(lbg_block b, const lbg_fluid* fluid, const lbg_box* range);
/* Several boxes in one launch (the 6 boundary_shell boxes, field.cpp:55-72). */
lbg_status lbg_sweep_boxes(lbg_block b, const lbg_fluid* fluid, const lbg_box* boxes, int n);
/* Periodic axes the sweep wraps in-kernel: for an axis the block spans completely (one
 * block along it), the pull of a population that would come from the ghost layer reads the
 * wrapped interior cell instead — the value fill_periodic_ghosts would have put there — so
 * the ghost fill for that axis is not needed. Bitwise identical interior results. */
lbg_status lbg_set_periodic_wrap(lbg_block b, const int wrap[3]);
/* Streaming layout of a plain-fluid block. LBG_STREAM_AB (default): the reference's two
 * buffers, pull sweep into dst, lbg_swap (field.hpp:36-78). LBG_STREAM_AA: in-place AA pattern
 * in ONE buffer (half the HBM; the other buffer is released): alternating steps read and write
 * each cell's own slots or its neighbours' (lbg_aa.cu), bitwise the same populations. Needs a
 * single periodic block with the in-kernel wrap on every axis (no BC, halo or coupling); each
 * step is lbg_sweep over the whole block + lbg_swap. lbg_download_src returns the double-buffer
 * src image in either phase; dst transfers, BCs, halos and box sweeps return LBG_INVALID;
 * moments and totals only after an even number of steps. Switching back re-allocates dst. */
enum { LBG_STREAM_AB = 0, LBG_STREAM_AA = 1 };
lbg_status lbg_set_streaming(lbg_block b, int mode);
/* Unfused pull stream (lbm.cpp:6-17), debug/tests. */
lbg_status lbg_stream(lbg_block b, const lbg_box* range);

/* fill_periodic_ghosts (boundary.cpp:98-137). full=1 copies all 19 q of all 26 regions
 * (bitwise identical src buffer); full=0 copies only the ghost slots a pull sweep reads. */
lbg_status lbg_fill_periodic(lbg_block b, const int periodic[3], int full);
/* apply_boundaries (boundary.cpp:32-96, 140-146). */
lbg_status lbg_apply_boundaries(lbg_block b, const lbg_face_bc faces[6], const int touches[6]);

/* ------------------------------------------------------------------ particle coupling */
/* SubBlockRegistry::build + build_fraction_field (psm.cpp:55-136), with the solid
 * velocities of set_solid_velocities (psm.cpp:138-169) following from these snapshots until
 * lbg_set_solid_velocities registers others: snapshots must be id-sorted; staged through
 * pinned memory and copied H2D on the block's side stream. `subdivisions` is accepted for
 * API parity (the device binning is finer and gives the same candidate order). */
lbg_status lbg_map(lbg_block b, const lbg_snapshot* snaps, int n, int subdivisions);
/* lbg_map into a second fraction field while the block keeps using the current one (its
 * sweeps, reductions and observers are unaffected): the next step's mapping can be issued as
 * soon as its inputs (ids, positions, radii) are final, overlapping host work. lbg_map_commit
 * makes the prepared field current (pointer swap); errors of the prepared mapping (overfull
 * cells) are reported by lbg_sync like lbg_map's. */
lbg_status lbg_map_prepare(lbg_block b, const lbg_snapshot* snaps, int n, int subdivisions);
lbg_status lbg_map_commit(lbg_block b);
/* set_solid_velocities (psm.cpp:138-169), replaces Simulation::phase_setu_inner's call
 * (sim.cpp:296-297). Uploads the (post velocity-sync) snapshots; the PSM sweep evaluates
 * u + omega x (c - x) per entry from them. If the list lost an id of the mapping list (or
 * the fraction field was uploaded by the caller), the per-entry walk runs here and counts
 * unknown ids, returning LBG_SYNC_ERROR itself (a synchronising call only then).
 * lbg_download_solid_velocity materialises v0/v1. */
lbg_status lbg_set_solid_velocities(lbg_block b, const lbg_snapshot* snaps, int n);
/* LBG_FORCE_SCRATCH (default) or LBG_FORCE_FUSED; takes effect at once. The fused per-particle
 * accumulators are sized and zeroed here, by lbg_map and by lbg_set_solid_velocities (the
 * snapshot list they are indexed by); a sweep in fused mode without them is LBG_INVALID. */
lbg_status lbg_set_force_mode(lbg_block b, int mode);
/* finalize_hydro_forces (psm.cpp:278-322): fills out[] id-sorted (one row per particle
 * with at least one entry), sets *n_out, clears the scratch. Blocks until done.
 * In LBG_FORCE_FUSED mode only LBG_REDUCE_FAST is available (comp terms are zero). */
lbg_status lbg_reduce_hydro(lbg_block b, int mode, lbg_hydro_partial* out, int capacity,
                            int* n_out);

/* Coupling fields (tests / parity; host arrays in the reference layouts above). */
lbg_status lbg_upload_fraction(lbg_block b, const uint8_t* count, const int* id0,
                               const int* id1, const double* b0, const double* b1,
                               const double* btot);
lbg_status lbg_download_fraction(lbg_block b, uint8_t* count, int* id0, int* id1, double* b0,
                                 double* b1, double* btot);
lbg_status lbg_upload_solid_velocity(lbg_block b, const double* v0, const double* v1);
lbg_status lbg_download_solid_velocity(lbg_block b, double* v0, double* v1);
lbg_status lbg_upload_scratch(lbg_block b, const double* m0, const double* m1);
lbg_status lbg_download_scratch(lbg_block b, double* m0, double* m1);

/* ------------------------------------------------------------------ sync / observers */
/* End-of-phase barrier: waits for the block's streams, returns and clears the error
 * counters; status LBG_NUMERIC_ERROR / LBG_SYNC_ERROR when any is nonzero. */
lbg_status lbg_sync(lbg_block b, lbg_errors* out);
/* total_mass / total_momentum of the src interior (lbm.cpp:69-93), Neumaier-compensated
 * per block of cells, then combined in fixed order (deterministic, not bitwise). */
lbg_status lbg_total_mass(lbg_block b, double* out);
lbg_status lbg_total_momentum(lbg_block b, double out[3]);
/* The fluid part of io::sample_scalars (output.cpp:22-45), one device pass over the src
 * interior: out = {mass, momentum x, y, z (bare moment, lbm.cpp:82-93), fluid kinetic energy
 * sum 0.5 rho |u|^2 and max |u| with the observable u = m + f_ext/2 (lbm.hpp:55-63)}.
 * Compensated, deterministic for a given device; not bitwise equal to the serial order. */
lbg_status lbg_observe(lbg_block b, const double f_ext[3], double out[6]);
/* Per-cell moments of the src interior for observers and grid dumps, replacing the host
 * walks over the PDF field in lbm::cell_macroscopic / total_mass / total_momentum
 * (lbm.cpp:61-93) and io::sample_scalars / write_grid_dump (output.cpp:22-107).
 * out[c*S + 0..3] = {rho, mx, my, mz}: rho = sum f_q and m = sum f_q c_q in q order, bitwise
 * the reference's sums; the observable velocity is m / 1.0 + 0.5 * f_ext (lbm.hpp:62), done
 * by the caller. With with_frac, S = 5 and out[c*S + 4] = btot (0 for an uncoupled block,
 * as write_grid_dump prints). Cells c = (k*ny + j)*nx + i. `out`: host memory of
 * nx*ny*nz*S doubles (pinned is faster). Blocking; 32-40 B per cell cross PCIe instead of
 * the 152 B of the populations. */
lbg_status lbg_moments(lbg_block b, int with_frac, double* out);

/* ------------------------------------------------------------------ halo exchange */
/* Simulation::begin/complete_halo_exchange (sim.cpp:156-201) for a slab decomposition
 * along `axis` over `nranks` processes (one GPU each), NCCL send/recv on a dedicated comm
 * stream; `periodic` is the domain's periodic mask (ring along `axis`, ghost-ring wrap of
 * received planes along the others). lbg_comm_unique_id is called on rank 0 and broadcast
 * by the caller. */
lbg_status lbg_comm_unique_id(char out[128]);
lbg_status lbg_comm_init(lbg_block b, int nranks, int rank, const char id[128], int axis,
                         const int periodic[3]);
lbg_status lbg_comm_destroy(lbg_block b);
/* Post-collision src boundary planes -> neighbours (non-blocking, comm stream). */
lbg_status lbg_halo_begin(lbg_block b);
/* Ghost planes valid for the outer sweep; SyncError without a pending begin (sim.cpp:183). */
lbg_status lbg_halo_complete(lbg_block b);

/* Generic in-process halo slabs with the reference's exact semantics, for block layouts the
 * NCCL slab exchange does not cover (several blocks per process, 26 neighbours):
 * lbg_pack_slab copies all 19 q of source_slab(off) (sim.cpp:120-135) from src into `out`
 * in PdfSlab order (q-major, then k, j, i; sim.cpp:167-173); lbg_unpack_slab writes `in` into
 * ghost_region(dir) (sim.cpp:137-152, 186-197). `out`/`in` are host buffers of
 * 19 * slab-cells doubles; *n_out receives that count. Both block until done. */
lbg_status lbg_pack_slab(lbg_block b, const int off[3], double* out, long long capacity,
                         long long* n_out);
lbg_status lbg_unpack_slab(lbg_block b, const int dir[3], const double* in, long long n);
/* The same exchange without the host: lbg_halo_stage packs source_slab(off) of every listed
 * neighbour offset into device staging buffers (begin_halo_exchange, async); a receiver then
 * calls lbg_halo_fetch(dst, dir, src) for each of its neighbour entries (src block at offset
 * dir): src's staged source_slab(-dir) is copied device-to-device (peer copy over NVLink when
 * the blocks live on different GPUs) and unpacked into dst's ghost_region(dir). All 19 q,
 * identical values to the message-bus path. Staging buffers are reused: a new lbg_halo_stage
 * waits (stream order) for every fetch that read the previous staging, so callers may
 * pipeline steps without a host synchronisation. */
lbg_status lbg_halo_stage(lbg_block b, const int (*offs)[3], int n);
lbg_status lbg_halo_fetch(lbg_block dst, const int dir[3], lbg_block src);
/* complete_halo_exchange (sim.cpp:181-201) for all n neighbour entries of dst at once:
 * (dirs[t], srcs[t]) as in lbg_halo_fetch, one unpack launch (the ghost regions of distinct
 * directions are disjoint, so the order of the reference's loop does not matter). */
lbg_status lbg_halo_fetch_all(lbg_block dst, const int (*dirs)[3], const lbg_block* srcs, int n);

/* The halo pushed by its sender, for several blocks of one process on any GPUs (replaces
 * begin/complete_halo_exchange, sim.cpp:156-201, once the ghosts have been filled by one
 * lbg_halo_stage / lbg_halo_fetch_all exchange). lbg_halo_push_connect registers the block's
 * neighbours (offset, block; not itself) and enables peer access to their GPUs. After each
 * sweep of the whole block (before any lbg_swap), lbg_halo_push stores the post-collision
 * populations that stream out through each face (5 q per face cell) and edge (1 q per edge
 * cell) straight into the neighbours' next-step ghost cells — the only ghost slots a pull sweep
 * reads — on the block's comm stream (NVLink peer stores across GPUs; no staging, no unpack),
 * asynchronous to the caller. lbg_halo_push_wait, at the start of the next step, orders the
 * block's stream after its neighbours' pushes (complete_halo_exchange). Interior results are
 * bitwise those of the full 19-q exchange; ghost slots no sweep reads are not written. Steps
 * must be lockstep across the registered blocks (every block pushes once per step). */
lbg_status lbg_halo_push_connect(lbg_block b, const int (*offs)[3], const lbg_block* nbrs, int n);
lbg_status lbg_halo_push(lbg_block b);
lbg_status lbg_halo_push_wait(lbg_block b);

/* The slab halo fused into the outer sweep over NVLink peer memory (one process per GPU,
 * >= 2 ranks, plain-fluid blocks). lbg_p2p_handles exports 208 bytes per rank: CUDA IPC
 * handles (both PDF buffers + a flag word array) and the block's layout; the caller all-gathers
 * them (rank order) and passes them to lbg_p2p_connect, which returns LBG_INVALID unless both
 * slab neighbours have this block's dimensions (the remote stores use the local layout). After every rank's state is set and a host barrier,
 * lbg_p2p_prime fills the slab-axis ghost planes once from the neighbours. Then each step:
 * lbg_sweep (inner planes 1..n-2) -> lbg_sweep_outer_p2p (waits for the neighbours' previous
 * outer sweep, computes the two boundary planes and stores their outbound populations
 * directly into the neighbours' ghost planes, then publishes the step) -> lbg_swap. Replaces
 * lbg_halo_begin/complete (no pack, no NCCL, no unpack). */
lbg_status lbg_p2p_handles(lbg_block b, void* out, size_t* bytes);
lbg_status lbg_p2p_connect(lbg_block b, int nranks, int rank, const void* all_handles, int axis,
                           const int periodic[3]);
lbg_status lbg_p2p_prime(lbg_block b);
lbg_status lbg_sweep_outer_p2p(lbg_block b, const lbg_fluid* fluid);
lbg_status lbg_p2p_destroy(lbg_block b);

/* ------------------------------------------------------------------ instrumentation */
/* Per-category CUDA-event timing (perf::Category names); off by default. */
lbg_status lbg_set_timing(lbg_block b, int on);
/* Sums (and clears) the elapsed device ms per category since the last call. */
lbg_status lbg_timings(lbg_block b, double ms[LBG_NUM_CATS], long long launches[LBG_NUM_CATS]);
/* Kernels this library launched (all blocks, process-wide). */
long long lbg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LBG_H */
