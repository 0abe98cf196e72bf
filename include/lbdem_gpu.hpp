// SPDX-License-Identifier: Apache-2.0
//
// lbdem_gpu.hpp — C++ host side of the drop-in: the reference's operator API (namespaces
// lbdem::lbm / lbdem::psm, /root/reference/proj/include/lbdem) re-expressed over the C ABI
// of liblbg (lbg.h). Include it inside the reference build (it uses the reference's own
// types and exception classes); INTEGRATION.md shows the sim.cpp call sites it replaces.
//
//   reference                                   lbdem::gpu::DeviceBlock
//   BlockState::field/frac/svel/scratch ctor    DeviceBlock(device, box, coupling)
//   Simulation::initialize_fluid                initialize_fluid(rho, u)
//   PdfField::src() (host copy for observers)   download_src(PdfField&) / upload_src(const PdfField&)
//   begin/complete_halo_exchange slab loops     pack_slab(off, values) / unpack_slab(dir, values)
//   psm::SubBlockRegistry::build +
//     psm::build_fraction_field                 map(snapshots, subdivisions)
//   psm::set_solid_velocities                   set_solid_velocities(snapshots)
//   run_kernel -> {psm_,}collide_stream_*       sweep(params, range) / sweep_boxes(params, boxes)
//   lbm::apply_boundaries                       apply_boundaries(spec, touches)
//   lbm::fill_periodic_ghosts                   fill_periodic_ghosts(periodic)
//   PdfField::swap                              swap()
//   psm::finalize_hydro_forces                  finalize_hydro_forces()
//   end-of-operator throws                      sync()  (NumericError / SyncError, same texts)
#pragma once

#include <algorithm>
#include <array>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbdem/boundary.hpp"
#include "lbdem/errors.hpp"
#include "lbdem/field.hpp"
#include "lbdem/lbm.hpp"
#include "lbdem/psm.hpp"
#include "lbg.h"

namespace lbdem::gpu {

/// lbg_status -> the reference exception of the same meaning (errors.hpp:10-32).
inline void check(lbg_status s) {
    if (s == LBG_OK) return;
    const std::string msg = lbg_last_error();
    switch (s) {
        case LBG_CONFIG_ERROR: throw ConfigError(msg);
        case LBG_NUMERIC_ERROR: throw NumericError(msg);
        case LBG_SYNC_ERROR: throw SyncError(msg);
        case LBG_IO_ERROR: throw IoError(msg);
        default: throw std::runtime_error("liblbg: " + msg);
    }
}

inline lbg_box to_box(const CellBox& b) {
    return {{b.lo.x, b.lo.y, b.lo.z}, {b.hi.x, b.hi.y, b.hi.z}};
}

inline lbg_fluid to_fluid(const lbm::FluidParams& p) { return {p.tau, {p.f_ext.x, p.f_ext.y, p.f_ext.z}}; }

class DeviceBlock {
public:
    /// force_mode: LBG_FORCE_SCRATCH (reference semantics, bitwise partials) or
    /// LBG_FORCE_FUSED (force/torque summed inside the PSM kernel; tolerance-level partials).
    /// -1 reads LBDEM_GPU_FORCE=fused|scratch from the environment (default scratch).
    DeviceBlock(int device, const CellBox& box, bool coupling, int force_mode = -1) {
        const Vec3i d = box.hi - box.lo;
        const int lo[3] = {box.lo.x, box.lo.y, box.lo.z};
        const int dims[3] = {d.x, d.y, d.z};
        check(lbg_block_create(device, lo, dims, coupling ? 1 : 0, &b_));
        if (force_mode < 0) {
            const char* e = std::getenv("LBDEM_GPU_FORCE");
            force_mode = (e && std::string(e) == "fused") ? LBG_FORCE_FUSED : LBG_FORCE_SCRATCH;
        }
        if (coupling) check(lbg_set_force_mode(b_, force_mode));
        fused_ = coupling && force_mode == LBG_FORCE_FUSED;
    }
    ~DeviceBlock() { lbg_block_destroy(b_); }
    DeviceBlock(const DeviceBlock&) = delete;
    DeviceBlock& operator=(const DeviceBlock&) = delete;

    lbg_block handle() const { return b_; }

    void initialize_fluid(double rho, const Vec3& u) {
        const double uu[3] = {u.x, u.y, u.z};
        check(lbg_fill_equilibrium(b_, rho, uu));
    }
    /// PdfField host copy <-> device src buffer (reference idx() layout, ghosts included).
    void upload_src(const PdfField& f) { check(lbg_upload_src(b_, f.src(0))); }
    void download_src(PdfField& f) const { check(lbg_download_src(b_, f.src(0))); }

    /// FractionField host copy (observers such as Simulation::fraction_at).
    void download_fraction(FractionField& f) const {
        check(lbg_download_fraction(b_, f.count.data(), f.id0.data(), f.id1.data(), f.b0.data(),
                                    f.b1.data(), f.btot.data()));
    }

    /// Per-cell {rho, mx, my, mz, btot} (lbg_moments), the input of the observers below.
    void moments(std::vector<double>& out) const {
        int dims[3];
        check(lbg_block_info(b_, dims, nullptr, nullptr, nullptr));
        out.resize(static_cast<std::size_t>(dims[0]) * dims[1] * dims[2] * 5);
        check(lbg_moments(b_, 1, out.data()));
    }

    void pack_slab(const Vec3i& off, std::vector<double>& values) const {
        long long n = 0;
        const int o[3] = {off.x, off.y, off.z};
        long long cells = 1;
        int dims[3];
        check(lbg_block_info(b_, dims, nullptr, nullptr, nullptr));
        for (int a = 0; a < 3; ++a) cells *= o[a] != 0 ? 1 : dims[a];
        values.resize(static_cast<std::size_t>(cells) * lbm::kQ);
        check(lbg_pack_slab(b_, o, values.data(), static_cast<long long>(values.size()), &n));
    }
    void unpack_slab(const Vec3i& dir, const std::vector<double>& values) {
        const int d[3] = {dir.x, dir.y, dir.z};
        check(lbg_unpack_slab(b_, d, values.data(), static_cast<long long>(values.size())));
    }

    /// Device-side halo (no host staging): stage this block's source slabs for its neighbour
    /// offsets (begin_halo_exchange), then fetch a neighbour's slab into a ghost region.
    void stage_slabs(const std::vector<Vec3i>& offsets) {
        std::vector<std::array<int, 3>> o;
        for (const Vec3i& v : offsets) o.push_back({v.x, v.y, v.z});
        check(lbg_halo_stage(b_, reinterpret_cast<const int(*)[3]>(o.data()), static_cast<int>(o.size())));
    }
    void fetch_slab(const Vec3i& dir, const DeviceBlock& from) {
        const int d[3] = {dir.x, dir.y, dir.z};
        check(lbg_halo_fetch(b_, d, from.b_));
    }
    /// complete_halo_exchange for all neighbour entries (dir, source block) in one launch
    void fetch_slabs(const std::vector<std::pair<Vec3i, const DeviceBlock*>>& from) {
        std::vector<std::array<int, 3>> d;
        std::vector<lbg_block> s;
        for (const auto& [v, blk] : from) {
            d.push_back({v.x, v.y, v.z});
            s.push_back(blk->b_);
        }
        check(lbg_halo_fetch_all(b_, reinterpret_cast<const int(*)[3]>(d.data()), s.data(),
                                 static_cast<int>(s.size())));
    }

    /// Sender-pushed halo (lbg_halo_push*): the neighbours this block pushes into; then per
    /// step push_halo() after the whole-block sweep and push_wait() before the next one.
    void push_connect(const std::vector<std::pair<Vec3i, const DeviceBlock*>>& to) {
        std::vector<std::array<int, 3>> d;
        std::vector<lbg_block> s;
        for (const auto& [v, blk] : to) {
            d.push_back({v.x, v.y, v.z});
            s.push_back(blk->b_);
        }
        check(lbg_halo_push_connect(b_, reinterpret_cast<const int(*)[3]>(d.data()), s.data(),
                                    static_cast<int>(s.size())));
    }
    void push_halo() { check(lbg_halo_push(b_)); }
    void push_wait() { check(lbg_halo_push_wait(b_)); }

    void map(const std::vector<psm::ParticleSnapshot>& snaps, int subdivisions) {
        to_c(snaps);
        check(lbg_map(b_, cs_.data(), static_cast<int>(cs_.size()), subdivisions));
    }
    /// the next step's mapping into the shadow fraction field (lbg_map_prepare) / make it current
    void map_prepare(const std::vector<psm::ParticleSnapshot>& snaps, int subdivisions) {
        std::vector<lbg_snapshot> c(snaps.size());
        for (std::size_t i = 0; i < snaps.size(); ++i) {
            const auto& s = snaps[i];
            c[i] = lbg_snapshot{s.id, 0, {s.x.x, s.x.y, s.x.z}, s.r, s.f_r,
                                {s.u.x, s.u.y, s.u.z}, {s.omega.x, s.omega.y, s.omega.z}};
        }
        check(lbg_map_prepare(b_, c.data(), static_cast<int>(c.size()), subdivisions));
    }
    void map_commit() { check(lbg_map_commit(b_)); }
    void set_solid_velocities(const std::vector<psm::ParticleSnapshot>& snaps) {
        to_c(snaps);
        check(lbg_set_solid_velocities(b_, cs_.data(), static_cast<int>(cs_.size())));
    }

    void sweep(const lbm::FluidParams& p, const CellBox& range) {
        const lbg_fluid f = to_fluid(p);
        const lbg_box r = to_box(range);
        check(lbg_sweep(b_, &f, &r));
    }
    void sweep_boxes(const lbm::FluidParams& p, const std::vector<CellBox>& boxes) {
        const lbg_fluid f = to_fluid(p);
        std::vector<lbg_box> bs;
        for (const CellBox& b : boxes) bs.push_back(to_box(b));
        for (std::size_t s = 0; s < bs.size(); s += 8)
            check(lbg_sweep_boxes(b_, &f, bs.data() + s, static_cast<int>(std::min<std::size_t>(8, bs.size() - s))));
    }
    void apply_boundaries(const lbm::BcSpec& spec, const std::array<bool, 6>& touches) {
        lbg_face_bc faces[6];
        int t[6];
        for (int f = 0; f < 6; ++f) {
            faces[f].kind = static_cast<int>(spec.faces[f].kind);
            faces[f].pad_ = 0;
            faces[f].u_wall[0] = spec.faces[f].u_wall.x;
            faces[f].u_wall[1] = spec.faces[f].u_wall.y;
            faces[f].u_wall[2] = spec.faces[f].u_wall.z;
            faces[f].rho = spec.faces[f].rho;
            t[f] = touches[f] ? 1 : 0;
        }
        check(lbg_apply_boundaries(b_, faces, t));
    }
    void fill_periodic_ghosts(const std::array<bool, 3>& periodic, bool full = true) {
        const int p[3] = {periodic[0], periodic[1], periodic[2]};
        check(lbg_fill_periodic(b_, p, full ? 1 : 0));
    }
    void swap() { check(lbg_swap(b_)); }
    /// Simulation::run(steps) (sim.cpp:702-704) of a periodic fluid block on a host PdfField in
    /// the reference layout (`host`, pinned for overlap), in place: lbg_run_host's pipelined
    /// upload / sweeps / download; NumericError as the reference's end-of-sweep check.
    void run_host(const lbm::FluidParams& p, double* host, int steps, int slab_planes = 0) {
        const lbg_fluid f = to_fluid(p);
        check(lbg_run_host(b_, &f, host, steps, slab_planes, nullptr));
    }

    std::vector<psm::HydroPartial> finalize_hydro_forces(int mode = -1) {
        if (mode < 0) mode = fused_ ? LBG_REDUCE_FAST : LBG_REDUCE_PARITY;
        // the raw partials buffer persists across steps (no 1-MB value-initialised allocation
        // per call at 10^4 particles)
        if (red_out_.size() < cs_.size() + 1) red_out_.resize(cs_.size() + 1);
        lbg_hydro_partial* out = red_out_.data();
        int n = 0;
        check(lbg_reduce_hydro(b_, mode, out, static_cast<int>(red_out_.size()), &n));
        std::vector<psm::HydroPartial> parts(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            parts[i].id = out[i].id;
            parts[i].f = {out[i].f[0], out[i].f[1], out[i].f[2]};
            parts[i].f_comp = {out[i].f_comp[0], out[i].f_comp[1], out[i].f_comp[2]};
            parts[i].t = {out[i].t[0], out[i].t[1], out[i].t[2]};
            parts[i].t_comp = {out[i].t_comp[0], out[i].t_comp[1], out[i].t_comp[2]};
        }
        return parts;
    }

    /// End-of-operator check: throws the reference exception the CPU operator would have.
    lbg_errors sync() {
        lbg_errors e{};
        check(lbg_sync(b_, &e));
        return e;
    }

private:
    void to_c(const std::vector<psm::ParticleSnapshot>& snaps) {
        cs_.resize(snaps.size());
        for (std::size_t i = 0; i < snaps.size(); ++i) {
            const auto& s = snaps[i];
            cs_[i] = lbg_snapshot{s.id, 0, {s.x.x, s.x.y, s.x.z}, s.r, s.f_r,
                                  {s.u.x, s.u.y, s.u.z}, {s.omega.x, s.omega.y, s.omega.z}};
        }
    }

    lbg_block b_ = nullptr;
    bool fused_ = false;
    std::vector<lbg_snapshot> cs_;
    std::vector<lbg_hydro_partial> red_out_;
};

}  // namespace lbdem::gpu
