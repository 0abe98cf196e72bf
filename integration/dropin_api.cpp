// SPDX-License-Identifier: Apache-2.0
//
// Scenario-runner C API of the drop-in build (the reference Simulation with its GPU-side
// operators on liblbg): what a ctypes / cgo / JNI binding of the reference's run loop
// would call. Config JSON in (io::parse_config, config.cpp:116-244), steps, observers and
// the reference's per-category TimingReport (perf.hpp:17-26) out.
// Status codes as lbg.h: 0 ok, 1 ConfigError, 2 NumericError, 3 SyncError, 4 IoError, 5 other.

#include <cmath>
#include <memory>
#include <string>
#include <vector>

#include "lbdem/config.hpp"
#include "lbdem/errors.hpp"
#include "lbdem/output.hpp"
#include "lbdem/perf.hpp"
#include "lbdem/scenario.hpp"
#include "lbdem/sim.hpp"
#include "lbdem_gpu.hpp"

using namespace lbdem;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const NumericError& e) {
        g_err = e.what();
        return 2;
    } catch (const SyncError& e) {
        g_err = e.what();
        return 3;
    } catch (const IoError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

struct Run {
    io::ScenarioConfig cfg;
    std::unique_ptr<Simulation> sim;
};

Run* R(void* h) { return static_cast<Run*>(h); }

}  // namespace

extern "C" {

const char* dropin_last_error() { return g_err.c_str(); }

void* dropin_sim_create(const char* json_text) {
    auto* r = new Run;
    if (guarded([&] {
            r->cfg = io::parse_config(json_text);
            r->sim = io::build_scenario(r->cfg);
        }) != 0) {
        delete r;
        return nullptr;
    }
    return r;
}

void dropin_sim_destroy(void* h) { delete R(h); }

int dropin_sim_run(void* h, long steps) {
    return guarded([&] { R(h)->sim->run(steps); });
}

// Simulation::add_particles (sim.cpp:67-94) with rows {id, x, y, z, r, m}: test scenarios
// the presets cannot make (e.g. three spheres sharing cells)
int dropin_sim_add_particles(void* h, int n, const double* rows) {
    return guarded([&] {
        std::vector<dem::Particle> ps(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            const double* r = rows + 6 * i;
            ps[i].id = static_cast<int>(r[0]);
            ps[i].x = {r[1], r[2], r[3]};
            ps[i].r = r[4];
            ps[i].m = r[5];
        }
        R(h)->sim->add_particles(ps);
    });
}

long dropin_sim_cells(void* h) {
    const Vec3i d = R(h)->cfg.domain;
    return static_cast<long>(d.x) * d.y * d.z;
}

int dropin_sim_num_particles(void* h) { return static_cast<int>(R(h)->sim->gather_particles().size()); }

/// Per particle: id, x, u, w, f_hydro, t_hydro (16 doubles per row, as oracle/ref_shim.cpp).
void dropin_sim_particles(void* h, double* rows) {
    const auto ps = R(h)->sim->gather_particles();
    for (std::size_t i = 0; i < ps.size(); ++i) {
        double* r = rows + 16 * i;
        r[0] = ps[i].id;
        const Vec3* v[5] = {&ps[i].x, &ps[i].u, &ps[i].w, &ps[i].f_hydro, &ps[i].t_hydro};
        for (int a = 0; a < 5; ++a) {
            r[1 + 3 * a] = v[a]->x;
            r[2 + 3 * a] = v[a]->y;
            r[3 + 3 * a] = v[a]->z;
        }
    }
}

/// Interior PDFs, global lexicographic (k, j, i), q innermost.
void dropin_sim_pdfs(void* h, double* out) {
    auto& r = *R(h);
    const Vec3i D = r.cfg.domain;
    long n = 0;
    for (int k = 0; k < D.z; ++k)
        for (int j = 0; j < D.y; ++j)
            for (int i = 0; i < D.x; ++i)
                for (int q = 0; q < lbm::kQ; ++q) out[n++] = r.sim->pdf_at({i, j, k}, q);
}

double dropin_sim_mass(void* h) { return R(h)->sim->total_fluid_mass(); }

/// validation.cpp:46-63 shear-wave initial state, written on the host and uploaded.
int dropin_sim_shear_wave(void* h) {
    return guarded([&] {
        auto& r = *R(h);
        for (int b = 0; b < r.sim->num_blocks(); ++b) {
            BlockState& blk = r.sim->block(b);
            const Vec3i d = blk.dims();
            if (blk.field.nx() != d.x) throw ConfigError("shear-wave init needs LBDEM_GPU_HOST_MIRROR=1");
            for (int k = 0; k < d.z; ++k)
                for (int j = 0; j < d.y; ++j)
                    for (int i = 0; i < d.x; ++i) {
                        const double gx = blk.box.lo.x + i + 0.5;
                        const double gy = blk.box.lo.y + j + 0.5;
                        const double gz = blk.box.lo.z + k + 0.5;
                        const Vec3 u{0.02 * std::sin(2.0 * dem::kPi * gy / r.cfg.domain.y),
                                     0.015 * std::cos(2.0 * dem::kPi * gz / r.cfg.domain.z),
                                     0.01 * std::sin(2.0 * dem::kPi * gx / r.cfg.domain.x)};
                        const auto feq = lbm::equilibrium(1.0, u);
                        const long base = blk.field.idx(i, j, k);
                        for (int q = 0; q < lbm::kQ; ++q) blk.field.src(q)[base] = feq[q];
                    }
            blk.dev->upload_src(blk.field);
            blk.moments_stale = true;
        }
    });
}

/// io::sample_scalars (output.cpp:22-61): step, mass, momentum xyz, fluid KE, particle KE,
/// min gap, max |u| — through the drop-in observers (device moments).
int dropin_sim_observe(void* h, double out[9]) {
    return guarded([&] {
        const io::ScalarSample s = io::sample_scalars(*R(h)->sim);
        const double v[9] = {static_cast<double>(s.step), s.mass, s.momentum.x, s.momentum.y,
                             s.momentum.z, s.fluid_ke, s.particle_ke, s.min_gap, s.max_u};
        for (int a = 0; a < 9; ++a) out[a] = v[a];
    });
}

/// io::write_grid_dump (output.cpp:76-107) of the current state to `path`.
int dropin_sim_grid_dump(void* h, const char* path) {
    return guarded([&] { io::write_grid_dump(*R(h)->sim, path); });
}

void dropin_sim_reset_timers(void* h) { R(h)->sim->reset_timers(); }

/// Per-category seconds, max over workers (perf::TimingReport convention, perf.cpp:25-45).
void dropin_sim_timings(void* h, double out[8]) {
    const auto per = R(h)->sim->timings_per_worker();
    for (int c = 0; c < perf::kCategories && c < 8; ++c) {
        out[c] = 0.0;
        for (const auto& t : per) out[c] = std::max(out[c], t.seconds[c]);
    }
}

}  // extern "C"
