"""Builds the drop-in: the reference solver with its GPU-side operators served by liblbg.

This is what a maintainer of the reference does: the host program —
Simulation's phase structure, DEM, particle messaging, partial routing, config, scenarios —
stays the reference's own code, and the call sites of the fluid/coupling operators in
sim.cpp / the fields in sim.hpp's BlockState are pointed at lbdem::gpu::DeviceBlock
(include/lbdem_gpu.hpp). The edits are applied to copies of those files (and of output.cpp, whose observers read
device moments) in integration/_build/ (git-ignored; no reference source enters the repository); every other
reference source compiles unmodified from /root/reference.

    python integration/make_dropin.py      # -> integration/_build/liblbdem_dropin.so
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.environ.get("LBDEM_REF", "/root/reference/proj")
BUILD = os.path.join(HERE, "_build")

# (anchor in the reference file, replacement). Each edit names the reference lines it replaces.
SIM_HPP_EDITS = [
    # sim.hpp:12 — forward declaration of the device twin
    ('#include "lbdem/psm.hpp"\n',
     '#include "lbdem/psm.hpp"\n\nnamespace lbdem::gpu {\nclass DeviceBlock;\n}\n'),
    # sim.hpp:49 — BlockState gains its device twin (field/frac/svel/scratch live on the GPU)
    ("    bool halo_pending = false;\n",
     "    bool halo_pending = false;\n"
     "    std::shared_ptr<gpu::DeviceBlock> dev;  ///< liblbg block (drop-in)\n"
     "    mutable bool host_stale = false;        ///< host field copy behind the device\n"
     "    mutable std::vector<double> moments;    ///< device moments cache (observers)\n"
     "    mutable bool moments_stale = true;\n"
     "    bool outer_done = false;                ///< whole block swept in phase_setu_inner\n"
     "    bool push_connected = false;            ///< lbg_halo_push neighbours registered\n"
     "    bool push_ready = false;                ///< ghosts kept current by the neighbours' pushes\n"
     "    bool premapped = false;                 ///< next step's fraction field already mapped\n"
     "    std::vector<psm::ParticleSnapshot> premap;  ///< the snapshots it was mapped from\n"),
]

SIM_CPP_EDITS = [
    # includes + host-copy refresh used by the observers
    ("#include <set>\n",
     "#include <set>\n#include <cstdlib>\n#include <cstring>\n#include <limits>\n\n#include \"lbdem_gpu.hpp\"\n#include \"dropin_observe.hpp\"\n#include \"dropin_sched.hpp\"\n"),
    ("namespace lbdem {\n\nusing partition::MsgKind;",
     "namespace lbdem {\n\n"
     "namespace {\n"
     "/// Device of block `id`: LBDEM_GPU_DEVICE (default 0), or with LBDEM_GPU_SPREAD=1 the\n"
     "/// blocks are dealt over all visible GPUs (one worker thread per block): consecutive runs\n"
     "/// of LBDEM_GPU_BLOCKS_PER_DEVICE (default 1) block ids per GPU, so neighbouring slabs of\n"
     "/// one GPU exchange their halo on the device and the host DEM has more workers.\n"
     "int gpu_device(int id) {\n"
     "    const char* s = std::getenv(\"LBDEM_GPU_SPREAD\");\n"
     "    if (s && std::atoi(s) != 0) {\n"
     "        const char* bp = std::getenv(\"LBDEM_GPU_BLOCKS_PER_DEVICE\");\n"
     "        const int per = bp ? std::max(1, std::atoi(bp)) : 1;\n"
     "        return (id / per) % std::max(1, lbg_device_count());\n"
     "    }\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_DEVICE\");\n"
     "    return e ? std::atoi(e) : 0;\n"
     "}\n"
     "/// LBDEM_GPU_HOST_MIRROR=0: no host PdfField/coupling copies (large runs; observers off).\n"
     "bool host_mirror() {\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_HOST_MIRROR\");\n"
     "    return !(e && std::atoi(e) == 0);\n"
     "}\n"
     "int mirror_dim(int d) { return host_mirror() ? d : 1; }\n"
     "/// PDF halo (LBDEM_GPU_HALO): push (default) - after the first step every block stores the\n"
     "/// populations leaving through its faces/edges into its neighbours' next-step ghosts right\n"
     "/// after its sweep (lbg_halo_push, 5 q per face cell, peer stores across GPUs); stage - the\n"
     "/// 19-q source slabs staged and fetched device to device every step; host - the MessageBus.\n"
     "int halo_mode() {\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_HALO\");\n"
     "    if (e && std::string(e) == \"host\") return 0;\n"
     "    if (e && std::string(e) == \"stage\") return 1;\n"
     "    return 2;\n"
     "}\n"
     "bool device_halo() { return halo_mode() != 0; }\n"
     "/// LBDEM_GPU_SWEEP=split: the reference's inner sweep / halo / BCs / outer-shell sweep;\n"
     "/// default one sweep of the whole block in phase_setu_inner after the halo and BCs (the\n"
     "/// halo messages were posted in phase_post_and_map; the inner sweep reads no ghost, so\n"
     "/// the results are identical) - no strided x-face shell sweep.\n"
     "bool full_sweep() {\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_SWEEP\");\n"
     "    return !(e && std::string(e) == \"split\");\n"
     "}\n"
     "/// the pushed halo needs the whole-block sweep (it follows the only sweep of a step)\n"
     "bool push_halo() { return halo_mode() == 2 && full_sweep(); }\n"
     "/// LBDEM_GPU_PREMAP=1: the next step's fraction field is mapped as soon as its inputs are\n"
     "/// final - in the last sub-cycle, right\n"
     "/// after the particle sync that fixes positions (sub_integrate_and_sync) and the block's\n"
     "/// particle/ghost membership (apply_particle_sync) - so the device mapping runs under the\n"
     "/// rest of that sub-cycle's host DEM (PAPER.md:576-583), into the block's second fraction\n"
     "/// field (observers after the step still see this step's). phase_post_and_map commits it\n"
     "/// when the snapshots it builds have the same ids, positions and radii (what the mapping\n"
     "/// reads), else maps as usual. Off by default: on config 3 it did not shorten the step\n"
     "/// (profiles/r02_premap.txt); the default maps in phase_post_and_map like the reference.\n"
     "bool premap_on() {\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_PREMAP\");\n"
     "    return e && std::atoi(e) != 0;\n"
     "}\n"
     "bool same_geometry(const std::vector<psm::ParticleSnapshot>& a,\n"
     "                   const std::vector<psm::ParticleSnapshot>& b) {\n"
     "    if (a.size() != b.size()) return false;\n"
     "    for (std::size_t i = 0; i < a.size(); ++i)\n"
     "        if (a[i].id != b[i].id || std::memcmp(&a[i].x, &b[i].x, sizeof(Vec3)) != 0 ||\n"
     "            std::memcmp(&a[i].r, &b[i].r, sizeof(double)) != 0 ||\n"
     "            std::memcmp(&a[i].f_r, &b[i].f_r, sizeof(double)) != 0)\n"
     "            return false;\n"
     "    return true;\n"
     "}\n"
     "/// Observers read the host copies; refresh them from the device after a step.\n"
     "void refresh_host(const std::vector<std::unique_ptr<BlockState>>& blocks, bool coupling) {\n"
     "    if (!host_mirror()) throw std::runtime_error(\"observer needs LBDEM_GPU_HOST_MIRROR=1\");\n"
     "    for (const auto& b : blocks) {\n"
     "        if (!b->host_stale) continue;\n"
     "        BlockState& m = const_cast<BlockState&>(*b);\n"
     "        m.dev->download_src(m.field);\n"
     "        if (coupling) m.dev->download_fraction(m.frac);\n"
     "        m.host_stale = false;\n"
     "    }\n"
     "}\n"
     "/// LBDEM_GPU_FAST_SYNC=0: the reference's host particle-messaging code as written. Default:\n"
     "/// the same results (ids are unique and sorted, so every lookup, sort and patch below finds\n"
     "/// what the reference's finds) with the quadratic snapshot patch of apply_velocity_sync\n"
     "/// replaced by a binary search, apply_particle_sync's struct sort by an in-place key\n"
     "/// permutation into reused storage, and phase_apply_hydro's sort skipped when its input is\n"
     "/// already in (id, block) order, the partials' particle lookups done by a forward cursor,\n"
     "/// and the ghost-eligibility loops skipping particles deep inside the block (SURVEY\n"
     "/// 8(f)#3; profiles/r02_host_sync.txt).\n"
     "bool fast_sync() {\n"
     "    static const bool on = [] {\n"
     "        const char* e = std::getenv(\"LBDEM_GPU_FAST_SYNC\");\n"
     "        return !(e && std::atoi(e) == 0);\n"
     "    }();\n"
     "    return on;\n"
     "}\n"
     "/// apply_particle_sync's sort (ascending id; the reference checks uniqueness right after,\n"
     "/// so with unique ids the order is std::sort's): the (id, index) keys are sorted and the\n"
     "/// particles permuted in place along the cycles, one move each, no allocation\n"
     "void sort_by_id(std::vector<dem::Particle>& v) {\n"
     "    if (std::is_sorted(v.begin(), v.end(),\n"
     "                       [](const dem::Particle& a, const dem::Particle& b2) { return a.id < b2.id; }))\n"
     "        return;\n"
     "    thread_local std::vector<std::pair<int, int>> keys;\n"
     "    thread_local std::vector<unsigned char> done;\n"
     "    const std::size_t n = v.size();\n"
     "    keys.resize(n);\n"
     "    for (std::size_t i = 0; i < n; ++i) keys[i] = {v[i].id, static_cast<int>(i)};\n"
     "    std::sort(keys.begin(), keys.end());\n"
     "    done.assign(n, 0);\n"
     "    for (std::size_t i = 0; i < n; ++i) {\n"
     "        if (done[i]) continue;\n"
     "        done[i] = 1;\n"
     "        if (static_cast<std::size_t>(keys[i].second) == i) continue;\n"
     "        dem::Particle tmp = std::move(v[i]);\n"
     "        std::size_t j = i;\n"
     "        for (;;) {\n"
     "            const std::size_t src = static_cast<std::size_t>(keys[j].second);\n"
     "            done[j] = 1;\n"
     "            if (src == i) {\n"
     "                v[j] = std::move(tmp);\n"
     "                break;\n"
     "            }\n"
     "            v[j] = std::move(v[src]);\n"
     "            j = src;\n"
     "        }\n"
     "    }\n"
     "}\n"
     "/// blk.particle(id) for ascending ids (the partial lists of phase_outer_reduce and\n"
     "/// phase_apply_hydro): a forward cursor over the id-sorted particle list finds what the\n"
     "/// binary search finds without its cache-missing probes; any id below the last one asked\n"
     "/// falls back to the binary search\n"
     "struct ParticleCursor {\n"
     "    BlockState& blk;\n"
     "    std::size_t i = 0;\n"
     "    int last = std::numeric_limits<int>::min();\n"
     "    dem::Particle* operator()(int id) {\n"
     "        if (!fast_sync() || id < last) return blk.particle(id);\n"
     "        last = id;\n"
     "        auto& v = blk.particles;\n"
     "        while (i < v.size() && v[i].id < id) ++i;\n"
     "        return (i < v.size() && v[i].id == id) ? &v[i] : nullptr;\n"
     "    }\n"
     "};\n"
     "/// a particle of the block whose distance to every face of the block box exceeds its ghost\n"
     "/// reach (r + margin, with a 1e-9 relative guard far above rounding) is ghost-eligible for\n"
     "/// no other block: any other block's box lies outside this one, so ghost_eligible's d2 is at\n"
     "/// least that distance squared. The neighbour loops skip it (false for a particle outside).\n"
     "bool deep_inside(const dem::Particle& p, const CellBox& box, double margin) {\n"
     "    const double reach = p.r + margin;\n"
     "    double dmin = std::numeric_limits<double>::infinity();\n"
     "    for (int a = 0; a < 3; ++a) {\n"
     "        const double lo = box.lo[a], hi = box.hi[a];\n"
     "        if (!(p.x[a] >= lo && p.x[a] <= hi)) return false;\n"
     "        dmin = std::min(dmin, std::min(p.x[a] - lo, hi - p.x[a]));\n"
     "    }\n"
     "    return dmin > reach * (1.0 + 1e-9);\n"
     "}\n"
     "/// LBDEM_GPU_SPIN_PHASES=0: the reference's ThreadPoolScheduler as built by the scenario;\n"
     "/// default: the same contract with spin-published phases (dropin_sched.hpp)\n"
     "std::unique_ptr<partition::Scheduler> phase_scheduler(std::unique_ptr<partition::Scheduler> s) {\n"
     "    const char* e = std::getenv(\"LBDEM_GPU_SPIN_PHASES\");\n"
     "    if ((e && std::atoi(e) == 0) || !dynamic_cast<partition::ThreadPoolScheduler*>(s.get())) return s;\n"
     "    const char* us = std::getenv(\"LBDEM_GPU_SPIN_US\");  // spin budget before blocking (A/B)\n"
     "    const char* pin = std::getenv(\"LBDEM_GPU_PIN_STRIDE\");  // worker w -> CPU w * stride (A/B)\n"
     "    return std::make_unique<gpu::SpinPhaseScheduler>(s->workers(), us ? std::atoi(us) : 2000,\n"
     "                                                     pin ? std::atoi(pin) : 0);\n"
     "}\n"
     "/// apply_particle_sync's list reuses the storage of the list it replaced (per worker thread)\n"
     "thread_local std::vector<dem::Particle> particle_scratch;\n"
     "}  // namespace\n\n"
     "using partition::MsgKind;"),
    # sim.cpp:15-25 — BlockState ctor: optional host mirror, create the device block
    ("      field(box_.hi.x - box_.lo.x, box_.hi.y - box_.lo.y, box_.hi.z - box_.lo.z) {\n"
     "    if (coupling) {\n",
     "      field(mirror_dim(box_.hi.x - box_.lo.x), mirror_dim(box_.hi.y - box_.lo.y),\n"
     "            mirror_dim(box_.hi.z - box_.lo.z)) {\n"
     "    if (coupling && host_mirror()) {\n"),
    ("        scratch.resize(frac.cells());\n    }\n}\n",
     "        scratch.resize(frac.cells());\n    }\n"
     "    dev = std::make_shared<gpu::DeviceBlock>(gpu_device(id_), box_, coupling);\n}\n"),
    # sim.cpp:54-57 — initialize_fluid on the device too
    ("    for (auto& blk : blocks_) blk->field.fill_src(feq);\n",
     "    for (auto& blk : blocks_) {\n"
     "        if (host_mirror()) blk->field.fill_src(feq);\n"
     "        blk->dev->initialize_fluid(rho, u);\n"
     "        blk->moments_stale = true;\n"
     "    }\n"),
    # sim.cpp:156-158 — halo begin: stage the source slabs on the device (no host copy); the
    # message-bus path below stays available with LBDEM_GPU_HALO=host
    ("void Simulation::begin_halo_exchange(int b) {\n    BlockState& blk = *blocks_[b];\n",
     "void Simulation::begin_halo_exchange(int b) {\n    BlockState& blk = *blocks_[b];\n"
     "    if (device_halo()) {\n"
     "        // once pushing, only periodic self-neighbours still go through the staging\n"
     "        const bool pushed = push_halo() && blk.push_ready;\n"
     "        std::vector<Vec3i> offs;\n"
     "        for (const auto& n : decomp_.blocks[b].neighbors)\n"
     "            if (!(pushed && n.block != b)) offs.push_back(n.offset);\n"
     "        blk.dev->stage_slabs(offs);\n"
     "        blk.halo_pending = true;\n"
     "        return;\n"
     "    }\n"),
    # sim.cpp:181-186 — halo complete: each neighbour entry (s, o) fills ghost_region(o) with
    # s's staged source_slab(-o), device to device (peer copy across GPUs), all in one launch
    ("    if (!blk.halo_pending) throw SyncError(\"halo completion without a pending exchange\");\n",
     "    if (!blk.halo_pending) throw SyncError(\"halo completion without a pending exchange\");\n"
     "    if (device_halo()) {\n"
     "        const bool pushed = push_halo() && blk.push_ready;\n"
     "        std::vector<std::pair<Vec3i, const gpu::DeviceBlock*>> from;\n"
     "        for (const auto& n : decomp_.blocks[b].neighbors)\n"
     "            if (!(pushed && n.block != b)) from.emplace_back(n.offset, blocks_[n.block]->dev.get());\n"
     "        if (!from.empty()) blk.dev->fetch_slabs(from);  // all staged entries in one unpack launch\n"
     "        if (pushed) blk.dev->push_wait();  // the neighbours' pushes of the previous step\n"
     "        blk.halo_pending = false;\n"
     "        return;\n"
     "    }\n"),
    # sim.cpp:167-173 — pack the source slab from the device
    ("        for (int q = 0; q < lbm::kQ; ++q) {\n"
     "            const double* p = blk.field.src(q);\n"
     "            for (int k = src.lo.z; k < src.hi.z; ++k)\n"
     "                for (int j = src.lo.y; j < src.hi.y; ++j)\n"
     "                    for (int i = src.lo.x; i < src.hi.x; ++i)\n"
     "                        slab.values.push_back(p[blk.field.idx(i, j, k)]);\n"
     "        }\n",
     "        blk.dev->pack_slab(n.offset, slab.values);\n"),
    # sim.cpp:189-197 — unpack into the device ghost region
    ("            const CellBox dst = ghost_region(dims, slab.dir);\n"
     "            std::size_t v = 0;\n"
     "            for (int q = 0; q < lbm::kQ; ++q) {\n"
     "                double* p = blk.field.src(q);\n"
     "                for (int k = dst.lo.z; k < dst.hi.z; ++k)\n"
     "                    for (int j = dst.lo.y; j < dst.hi.y; ++j)\n"
     "                        for (int i = dst.lo.x; i < dst.hi.x; ++i)\n"
     "                            p[blk.field.idx(i, j, k)] = slab.values[v++];\n"
     "            }\n",
     "            (void)dims;\n"
     "            blk.dev->unpack_slab(slab.dir, slab.values);\n"),
    # sim.cpp:221-236 — run_kernel: the device sweep (plain or PSM per the block's coupling)
    ("    if (range.empty()) return;\n"
     "    if (params_.coupling) {\n"
     "        if (params_.kernels == KernelMode::openmp)\n"
     "            psm::psm_collide_stream_omp(blk.field, params_.fluid, blk.frac, blk.svel,\n"
     "                                        blk.scratch, range);\n"
     "        else\n"
     "            psm::psm_collide_stream_serial(blk.field, params_.fluid, blk.frac, blk.svel,\n"
     "                                           blk.scratch, range);\n"
     "    } else {\n"
     "        if (params_.kernels == KernelMode::openmp)\n"
     "            lbm::collide_stream_omp(blk.field, params_.fluid, range);\n"
     "        else\n"
     "            lbm::collide_stream_serial(blk.field, params_.fluid, range);\n"
     "    }\n",
     "    if (range.empty()) return;\n"
     "    blk.dev->sweep(params_.fluid, range);\n"),
    # sim.cpp:278-280 — registry + build_fraction_field -> device mapping
    ("        blk.registry.build(blk.box, blk.snapshots, params_.subdivisions);\n"
     "        psm::build_fraction_field(blk.frac, blk.box, blk.registry, blk.snapshots,\n"
     "                                  params_.kernels == KernelMode::openmp);\n",
     "        if (blk.premapped && same_geometry(blk.premap, blk.snapshots))\n"
     "            blk.dev->map_commit();  // mapped during the last sub-cycle\n"
     "        else\n"
     "            blk.dev->map(blk.snapshots, params_.subdivisions);\n"
     "        blk.premapped = false;\n"
     "        // no wait here: the mapping runs under post_velocity_sync, checked right after it\n"),
    # sim.cpp:282-285 - the mapping's end-of-operator check (overfull cells: NumericError, the
    # reference's text) once the velocity records are posted
    ("        ScopedTimer t(blk.timings, Category::kPdComm);\n"
     "        post_velocity_sync(blk);\n"
     "    }\n",
     "        ScopedTimer t(blk.timings, Category::kPdComm);\n"
     "        post_velocity_sync(blk);\n"
     "    }\n"
     "    if (params_.coupling) {\n"
     "        ScopedTimer t(blk.timings, Category::kMapping);\n"
     "        blk.dev->sync();\n"
     "    }\n"),
    # sim.cpp:623-628 - the next step's mapping issued once its inputs are final (premap_on())
    ("        ScopedTimer t(blk.timings, Category::kPdComm);\n"
     "        apply_particle_sync(blk, s);\n"
     "    }\n",
     "        ScopedTimer t(blk.timings, Category::kPdComm);\n"
     "        apply_particle_sync(blk, s);\n"
     "    }\n"
     "    if (params_.coupling && premap_on() && s == params_.dem.subcycles - 1) {\n"
     "        ScopedTimer t(blk.timings, Category::kMapping);\n"
     "        build_snapshots(blk);\n"
     "        blk.premap = blk.snapshots;\n"
     "        blk.dev->map_prepare(blk.premap, params_.subdivisions);  // asynchronous, shadow field\n"
     "        blk.premapped = true;\n"
     "    }\n"),
    # sim.cpp:296-297 — set_solid_velocities on the device (post velocity-sync snapshots):
    # an asynchronous snapshot upload the PSM sweep evaluates u + omega x (c - x) from; it
    # raises SyncError itself when the exact per-entry walk finds unknown ids, so no sync here
    ("        psm::set_solid_velocities(blk.svel, blk.frac, blk.box, blk.snapshots,\n"
     "                                  params_.kernels == KernelMode::openmp);\n",
     "        blk.dev->set_solid_velocities(blk.snapshots);\n"),
    # sim.cpp:299-303 — inner kernel + end-of-operator check; by default the whole block
    # (halo completion and BCs of sim.cpp:307-312 moved ahead of it, see full_sweep())
    ("    {\n"
     "        ScopedTimer t(blk.timings, Category::kPsm);\n"
     "        const Vec3i d = blk.dims();\n"
     "        run_kernel(blk, {{1, 1, 1}, {d.x - 1, d.y - 1, d.z - 1}});\n"
     "    }\n",
     "    const Vec3i d = blk.dims();\n"
     "    if (full_sweep()) {\n"
     "        {\n"
     "            ScopedTimer t(blk.timings, Category::kPsmComm);\n"
     "            complete_halo_exchange(b);\n"
     "        }\n"
     "        blk.dev->apply_boundaries(params_.bc, blk.domain_faces);\n"
     "        ScopedTimer t(blk.timings, Category::kPsm);\n"
     "        run_kernel(blk, {{0, 0, 0}, {d.x, d.y, d.z}});\n"
     "        if (device_halo() && push_halo()) {\n"
     "            // the next step's halo leaves now, overlapping everything until then\n"
     "            if (!blk.push_connected) {\n"
     "                std::vector<std::pair<Vec3i, const gpu::DeviceBlock*>> to;\n"
     "                for (const auto& n : decomp_.blocks[b].neighbors)\n"
     "                    if (n.block != b) to.emplace_back(n.offset, blocks_[n.block]->dev.get());\n"
     "                blk.dev->push_connect(to);\n"
     "                blk.push_connected = true;\n"
     "            }\n"
     "            blk.dev->push_halo();\n"
     "            blk.push_ready = true;\n"
     "        }\n"
     "        blk.dev->sync();\n"
     "        blk.outer_done = true;\n"
     "    } else {\n"
     "        ScopedTimer t(blk.timings, Category::kPsm);\n"
     "        run_kernel(blk, {{1, 1, 1}, {d.x - 1, d.y - 1, d.z - 1}});\n"
     "        blk.dev->sync();\n"
     "    }\n"),
    # sim.cpp:307-317 — halo completion, BCs, outer shell in one launch, swap (skipped
    # when phase_setu_inner swept the whole block)
    ("    {\n"
     "        ScopedTimer t(blk.timings, Category::kPsmComm);\n"
     "        complete_halo_exchange(b);\n"
     "    }\n"
     "    lbm::apply_boundaries(blk.field, params_.bc, blk.domain_faces);\n"
     "    {\n"
     "        ScopedTimer t(blk.timings, Category::kPsm);\n"
     "        for (const CellBox& box : boundary_shell(blk.dims())) run_kernel(blk, box);\n"
     "    }\n"
     "    blk.field.swap();\n",
     "    if (!blk.outer_done) {\n"
     "        {\n"
     "            ScopedTimer t(blk.timings, Category::kPsmComm);\n"
     "            complete_halo_exchange(b);\n"
     "        }\n"
     "        blk.dev->apply_boundaries(params_.bc, blk.domain_faces);\n"
     "        ScopedTimer t(blk.timings, Category::kPsm);\n"
     "        blk.dev->sweep_boxes(params_.fluid, boundary_shell(blk.dims()));\n"
     "        blk.dev->sync();\n"
     "    }\n"
     "    blk.outer_done = false;\n"
     "    blk.dev->swap();\n"
     "    blk.host_stale = true;\n"
     "    blk.moments_stale = true;\n"),
    # sim.cpp:321 — finalize_hydro_forces on the device (PARITY: bitwise partials)
    ("    auto partials = psm::finalize_hydro_forces(blk.frac, blk.scratch, blk.box, blk.snapshots);\n",
     "    auto partials = blk.dev->finalize_hydro_forces();\n"),
    # sim.cpp:740-772 — observers: mass, momentum, macroscopic_at and fraction_at from the
    # device moments (dropin_observe.hpp, bitwise the reference's sums, no host mirror);
    # pdf_at still reads the refreshed host copy of the populations
    ("    for (const auto& blk : blocks_) m.add(lbm::total_mass(blk->field));\n",
     "    for (const auto& blk : blocks_) m.add(gpu::total_mass(*blk));\n"),
    ("    for (const auto& blk : blocks_) mom.add(lbm::total_momentum(blk->field));\n",
     "    for (const auto& blk : blocks_) mom.add(gpu::total_momentum(*blk));\n"),
    ("    lbm::cell_macroscopic(blk.field, params_.fluid.f_ext, cell.x - blk.box.lo.x,\n",
     "    gpu::cell_macroscopic(blk, params_.fluid.f_ext, cell.x - blk.box.lo.x,\n"),
    ("double Simulation::pdf_at(const Vec3i& cell, int q) const {\n",
     "double Simulation::pdf_at(const Vec3i& cell, int q) const {\n    refresh_host(blocks_, params_.coupling);\n"),
    ("    return blk.frac.btot[blk.frac.idx(cell.x - blk.box.lo.x, cell.y - blk.box.lo.y,\n"
     "                                      cell.z - blk.box.lo.z)];\n",
     "    return gpu::cell_fraction(blk, cell.x - blk.box.lo.x, cell.y - blk.box.lo.y,\n"
     "                              cell.z - blk.box.lo.z);\n"),
    # sim.cpp:249-266 - apply_velocity_sync: the snapshot patch by binary search (fast_sync())
    ("void Simulation::apply_velocity_sync(BlockState& blk) {\n",
     "void Simulation::apply_velocity_sync(BlockState& blk) {\n"
     "    const bool psorted = fast_sync() &&\n"
     "                         std::is_sorted(blk.snapshots.begin(), blk.snapshots.end(),\n"
     "                                        [](const psm::ParticleSnapshot& a, const psm::ParticleSnapshot& b2) {\n"
     "                                            return a.id < b2.id;\n"
     "                                        });\n"),
    ("            // Patch the kernel snapshot built before the sync arrived.\n"
     "            for (auto& s : blk.snapshots)\n"
     "                if (s.id == rec.id) {\n"
     "                    s.u = rec.u;\n"
     "                    s.omega = rec.w;\n"
     "                    break;\n"
     "                }\n",
     "            // Patch the kernel snapshot built before the sync arrived (ascending unique ids:\n"
     "            // the binary search finds the linear scan's match)\n"
     "            if (psorted) {\n"
     "                auto it = std::lower_bound(blk.snapshots.begin(), blk.snapshots.end(), rec.id,\n"
     "                                           [](const psm::ParticleSnapshot& s, int v) { return s.id < v; });\n"
     "                if (it != blk.snapshots.end() && it->id == rec.id) {\n"
     "                    it->u = rec.u;\n"
     "                    it->omega = rec.w;\n"
     "                }\n"
     "            } else {\n"
     "                for (auto& s : blk.snapshots)\n"
     "                    if (s.id == rec.id) {\n"
     "                        s.u = rec.u;\n"
     "                        s.omega = rec.w;\n"
     "                        break;\n"
     "                    }\n"
     "            }\n"),
    # sim.cpp:441-497 - apply_particle_sync: reused storage and the key-permutation sort
    ("    std::vector<dem::Particle> next;\n"
     "    next.reserve(blk.particles.size());\n",
     "    std::vector<dem::Particle> next;\n"
     "    if (fast_sync()) next = std::move(particle_scratch);\n"
     "    next.clear();\n"
     "    next.reserve(blk.particles.size());\n"),
    ("    std::sort(next.begin(), next.end(),\n"
     "              [](const dem::Particle& a, const dem::Particle& b2) { return a.id < b2.id; });\n",
     "    if (fast_sync())\n"
     "        sort_by_id(next);\n"
     "    else\n"
     "        std::sort(next.begin(), next.end(),\n"
     "                  [](const dem::Particle& a, const dem::Particle& b2) { return a.id < b2.id; });\n"),
    ("    blk.particles = std::move(next);\n"
     "    (void)s;\n",
     "    std::swap(blk.particles, next);\n"
     "    if (fast_sync()) particle_scratch = std::move(next);\n"
     "    (void)s;\n"),
    # sim.cpp:353-356 - phase_apply_hydro: no sort of a list already in (id, block) order
    ("    std::sort(all.begin(), all.end(), [](const auto& a, const auto& b2) {\n"
     "        if (a.second->id != b2.second->id) return a.second->id < b2.second->id;\n"
     "        return a.first < b2.first;\n"
     "    });\n",
     "    const auto by_id_src = [](const auto& a, const auto& b2) {\n"
     "        if (a.second->id != b2.second->id) return a.second->id < b2.second->id;\n"
     "        return a.first < b2.first;\n"
     "    };\n"
     "    if (!fast_sync() || !std::is_sorted(all.begin(), all.end(), by_id_src))\n"
     "        std::sort(all.begin(), all.end(), by_id_src);\n"),
    # sim.cpp:323-325 / 378-380 - the partials' particle lookups through the forward cursor
    ("    for (const psm::HydroPartial& p : partials) {\n"
     "        const dem::Particle* part = blk.particle(p.id);\n",
     "    ParticleCursor cursor{blk};\n"
     "    for (const psm::HydroPartial& p : partials) {\n"
     "        const dem::Particle* part = cursor(p.id);\n"),
    ("    std::size_t i = 0;\n"
     "    while (i < all.size()) {\n",
     "    ParticleCursor cursor{blk};\n"
     "    std::size_t i = 0;\n"
     "    while (i < all.size()) {\n"),
    ("        dem::Particle* part = blk.particle(id);\n"
     "        if (part == nullptr || part->ghost)\n",
     "        dem::Particle* part = cursor(id);\n"
     "        if (part == nullptr || part->ghost)\n"),
    # sim.cpp:322 / 347 - the partial lists sized once (fast_sync(); no regrowth copies)
    ("    blk.own_partials.clear();\n",
     "    blk.own_partials.clear();\n"
     "    if (fast_sync()) blk.own_partials.reserve(partials.size());\n"),
    ("    std::vector<std::pair<int, const psm::HydroPartial*>> all;\n",
     "    std::vector<std::pair<int, const psm::HydroPartial*>> all;\n"
     "    if (fast_sync()) all.reserve(blk.own_partials.size());\n"),
    # sim.cpp:243-246 / 433-437 - the ghost loops skip particles deep inside the block
    ("        for (const dem::Particle& p : blk.particles) {\n"
     "            if (p.ghost) continue;\n"
     "            if (ghost_eligible(p, nb)) per_dst[nb].push_back({p.id, p.u, p.w});\n",
     "        for (const dem::Particle& p : blk.particles) {\n"
     "            if (p.ghost) continue;\n"
     "            if (fast_sync() && deep_inside(p, blk.box, ghost_margin())) continue;\n"
     "            if (ghost_eligible(p, nb)) per_dst[nb].push_back({p.id, p.u, p.w});\n"),
    ("        const int owner = decomp_.block_of_position(p.x);\n"
     "\n"
     "        partition::StateRecord rec;\n",
     "        const int owner = decomp_.block_of_position(p.x);\n"
     "        // neither migrating nor a ghost anywhere: nothing to send\n"
     "        if (fast_sync() && owner == blk.id && deep_inside(p, blk.box, ghost_margin())) continue;\n"
     "\n"
     "        partition::StateRecord rec;\n"),
    # sim.cpp:39-44 - the phase scheduler (phase_scheduler(): spin-published phases)
    ("      scheduler_(std::move(scheduler)) {\n",
     "      scheduler_(phase_scheduler(std::move(scheduler))) {\n"),
]


# output.cpp:22-107 — sample_scalars and write_grid_dump read the device moments (the two
# per-cell macroscopic calls are the same line; (anchor, replacement, occurrences))
OUTPUT_CPP_EDITS = [
    ('#include "lbdem/output.hpp"\n',
     '#include "lbdem/output.hpp"\n#include "dropin_observe.hpp"\n', 1),
    ("lbm::cell_macroscopic(blk.field, sim.params().fluid.f_ext, i, j, k, rho, u);\n",
     "gpu::cell_macroscopic(blk, sim.params().fluid.f_ext, i, j, k, rho, u);\n", 2),
    ("sim.params().coupling ? blk.frac.btot[blk.frac.idx(i, j, k)] : 0.0;\n",
     "sim.params().coupling ? gpu::cell_fraction(blk, i, j, k) : 0.0;\n", 1),
]


def patch(src, edits, name):
    text = open(src).read()
    for e in edits:
        anchor, repl, n = e if len(e) == 3 else (*e, 1)
        if text.count(anchor) != n:
            sys.exit(f"{name}: anchor not found exactly {n}x:\n{anchor}")
        text = text.replace(anchor, repl)
    return text


def main():
    if not os.path.isdir(REF):
        if os.path.exists(os.path.join(BUILD, "liblbdem_dropin.so")):
            return 0
        sys.exit(f"reference sources not found at {REF}")
    os.makedirs(os.path.join(BUILD, "include", "lbdem"), exist_ok=True)
    os.makedirs(os.path.join(BUILD, "src"), exist_ok=True)
    hpp = patch(os.path.join(REF, "include/lbdem/sim.hpp"), SIM_HPP_EDITS, "sim.hpp")
    cpp = patch(os.path.join(REF, "src/sim.cpp"), SIM_CPP_EDITS, "sim.cpp")
    out = patch(os.path.join(REF, "src/output.cpp"), OUTPUT_CPP_EDITS, "output.cpp")
    for path, text in ((os.path.join(BUILD, "include/lbdem/sim.hpp"), hpp), (os.path.join(BUILD, "src/sim.cpp"), cpp),
                       (os.path.join(BUILD, "src/output.cpp"), out)):
        if not os.path.exists(path) or open(path).read() != text:
            open(path, "w").write(text)
    subprocess.check_call(["make", "-s", "-j8", "-C", HERE, f"REF={REF}"])
    return 0


if __name__ == "__main__":
    sys.exit(main())
