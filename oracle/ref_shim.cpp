// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled by oracle/Makefile into oracle/_ref/liblbdem_ref.so). It exists so the
// Python tests and bench.py's cpu_baseline / `--impl reference` leg can drive the
// reference's own operators (lbm.cpp, psm.cpp, boundary.cpp, sim.cpp) on raw
// arrays. Only tests/, __graft_entry__.smoke() and bench.py's reference leg may
// load the resulting library; the product path (paper_2303_11811_b200/) never does.
//
// Status codes mirror include/lbg.h: 0 ok, 1 ConfigError, 2 NumericError,
// 3 SyncError, 4 IoError, 5 other.

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "lbdem/boundary.hpp"
#include "lbdem/config.hpp"
#include "lbdem/errors.hpp"
#include "lbdem/field.hpp"
#include "lbdem/lbm.hpp"
#include "lbdem/output.hpp"
#include "lbdem/perf.hpp"
#include "lbdem/psm.hpp"
#include "lbdem/scenario.hpp"
#include "lbdem/sim.hpp"

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

struct RefBlock {
    CellBox box;
    PdfField field;
    FractionField frac;
    SolidVelocityField svel;
    CellMomentumScratch scratch;
    std::vector<psm::ParticleSnapshot> snaps;
    psm::SubBlockRegistry registry;

    RefBlock(const Vec3i& lo, const Vec3i& d)
        : box{lo, lo + d}, field(d.x, d.y, d.z), frac(d.x, d.y, d.z) {
        svel.resize(frac.cells());
        scratch.resize(frac.cells());
    }
};

RefBlock* B(void* h) { return static_cast<RefBlock*>(h); }

lbm::BcSpec make_bc(const int* kinds, const double* uwall, const double* rho) {
    lbm::BcSpec spec;
    for (int f = 0; f < 6; ++f) {
        spec.faces[f].kind = static_cast<lbm::BcKind>(kinds[f]);
        spec.faces[f].u_wall = {uwall[3 * f], uwall[3 * f + 1], uwall[3 * f + 2]};
        spec.faces[f].rho = rho[f];
    }
    return spec;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

// ---------------------------------------------------------------- block ops
void* ref_block_create(const int lo[3], const int dims[3]) {
    return new RefBlock({lo[0], lo[1], lo[2]}, {dims[0], dims[1], dims[2]});
}
void ref_block_destroy(void* h) { delete B(h); }
long ref_alloc_cells(void* h) { return B(h)->field.alloc_cells(); }

void ref_get_src(void* h, double* out) {
    auto& f = B(h)->field;
    for (int q = 0; q < lbm::kQ; ++q)
        std::memcpy(out + q * f.alloc_cells(), f.src(q), sizeof(double) * f.alloc_cells());
}
void ref_set_src(void* h, const double* in) {
    auto& f = B(h)->field;
    for (int q = 0; q < lbm::kQ; ++q)
        std::memcpy(f.src(q), in + q * f.alloc_cells(), sizeof(double) * f.alloc_cells());
}
void ref_get_dst(void* h, double* out) {
    auto& f = B(h)->field;
    for (int q = 0; q < lbm::kQ; ++q)
        std::memcpy(out + q * f.alloc_cells(), f.dst(q), sizeof(double) * f.alloc_cells());
}
void ref_set_dst(void* h, const double* in) {
    auto& f = B(h)->field;
    for (int q = 0; q < lbm::kQ; ++q)
        std::memcpy(f.dst(q), in + q * f.alloc_cells(), sizeof(double) * f.alloc_cells());
}
void ref_swap(void* h) { B(h)->field.swap(); }

int ref_fill_periodic(void* h, const int periodic[3]) {
    return guarded([&] {
        lbm::fill_periodic_ghosts(B(h)->field, {periodic[0] != 0, periodic[1] != 0, periodic[2] != 0});
    });
}

int ref_apply_boundaries(void* h, const int kinds[6], const double uwall[18], const double rho[6],
                         const int touches[6]) {
    return guarded([&] {
        const auto spec = make_bc(kinds, uwall, rho);
        std::array<bool, 6> t{};
        for (int f = 0; f < 6; ++f) t[f] = touches[f] != 0;
        lbm::apply_boundaries(B(h)->field, spec, t);
    });
}

int ref_sweep(void* h, double tau, const double fext[3], const int lo[3], const int hi[3],
              int coupling, int omp) {
    return guarded([&] {
        lbm::FluidParams p;
        p.tau = tau;
        p.f_ext = {fext[0], fext[1], fext[2]};
        const CellBox r{{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}};
        RefBlock& b = *B(h);
        if (coupling) {
            if (omp)
                psm::psm_collide_stream_omp(b.field, p, b.frac, b.svel, b.scratch, r);
            else
                psm::psm_collide_stream_serial(b.field, p, b.frac, b.svel, b.scratch, r);
        } else {
            if (omp)
                lbm::collide_stream_omp(b.field, p, r);
            else
                lbm::collide_stream_serial(b.field, p, r);
        }
    });
}

int ref_stream(void* h, const int lo[3], const int hi[3]) {
    return guarded([&] {
        lbm::stream(B(h)->field, {{lo[0], lo[1], lo[2]}, {hi[0], hi[1], hi[2]}});
    });
}

void ref_equilibrium(double rho, const double u[3], double feq[19]) {
    const auto f = lbm::equilibrium(rho, {u[0], u[1], u[2]});
    for (int q = 0; q < lbm::kQ; ++q) feq[q] = f[q];
}

int ref_total_mass(void* h, double* out) {
    return guarded([&] { *out = lbm::total_mass(B(h)->field); });
}
int ref_total_momentum(void* h, double out[3]) {
    return guarded([&] {
        const Vec3 m = lbm::total_momentum(B(h)->field);
        out[0] = m.x;
        out[1] = m.y;
        out[2] = m.z;
    });
}

// ------------------------------------------------------------- PSM coupling
int ref_f_of_r(double r, double* out) {
    return guarded([&] { *out = psm::f_of_r(r); });
}
double ref_sphere_volume(double r) { return psm::sphere_over_unit_square_volume(r); }

void ref_set_snapshots(void* h, int n, const int* ids, const double* x, const double* r,
                       const double* fr, const double* u, const double* w) {
    auto& s = B(h)->snaps;
    s.assign(n, {});
    for (int i = 0; i < n; ++i) {
        s[i].id = ids[i];
        s[i].x = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
        s[i].r = r[i];
        s[i].f_r = fr[i];
        s[i].u = {u[3 * i], u[3 * i + 1], u[3 * i + 2]};
        s[i].omega = {w[3 * i], w[3 * i + 1], w[3 * i + 2]};
    }
}

int ref_map(void* h, int subdivisions, int omp) {
    return guarded([&] {
        RefBlock& b = *B(h);
        b.registry.build(b.box, b.snaps, subdivisions);
        psm::build_fraction_field(b.frac, b.box, b.registry, b.snaps, omp != 0);
    });
}

int ref_set_u(void* h, int omp) {
    return guarded([&] {
        RefBlock& b = *B(h);
        psm::set_solid_velocities(b.svel, b.frac, b.box, b.snaps, omp != 0);
    });
}

long ref_frac_cells(void* h) { return B(h)->frac.cells(); }

void ref_get_fraction(void* h, std::uint8_t* count, int* id0, int* id1, double* b0, double* b1,
                      double* btot) {
    const auto& f = B(h)->frac;
    const long n = f.cells();
    std::memcpy(count, f.count.data(), n);
    std::memcpy(id0, f.id0.data(), n * sizeof(int));
    std::memcpy(id1, f.id1.data(), n * sizeof(int));
    std::memcpy(b0, f.b0.data(), n * sizeof(double));
    std::memcpy(b1, f.b1.data(), n * sizeof(double));
    std::memcpy(btot, f.btot.data(), n * sizeof(double));
}

void ref_set_fraction(void* h, const std::uint8_t* count, const int* id0, const int* id1,
                      const double* b0, const double* b1, const double* btot) {
    auto& f = B(h)->frac;
    const long n = f.cells();
    std::memcpy(f.count.data(), count, n);
    std::memcpy(f.id0.data(), id0, n * sizeof(int));
    std::memcpy(f.id1.data(), id1, n * sizeof(int));
    std::memcpy(f.b0.data(), b0, n * sizeof(double));
    std::memcpy(f.b1.data(), b1, n * sizeof(double));
    std::memcpy(f.btot.data(), btot, n * sizeof(double));
}

static void get_vec3s(const std::vector<Vec3>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[3 * i] = v[i].x;
        out[3 * i + 1] = v[i].y;
        out[3 * i + 2] = v[i].z;
    }
}
static void set_vec3s(std::vector<Vec3>& v, const double* in) {
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = {in[3 * i], in[3 * i + 1], in[3 * i + 2]};
}

void ref_get_svel(void* h, double* v0, double* v1) {
    get_vec3s(B(h)->svel.v0, v0);
    get_vec3s(B(h)->svel.v1, v1);
}
void ref_set_svel(void* h, const double* v0, const double* v1) {
    set_vec3s(B(h)->svel.v0, v0);
    set_vec3s(B(h)->svel.v1, v1);
}
void ref_get_scratch(void* h, double* m0, double* m1) {
    get_vec3s(B(h)->scratch.m0, m0);
    get_vec3s(B(h)->scratch.m1, m1);
}
void ref_set_scratch(void* h, const double* m0, const double* m1) {
    set_vec3s(B(h)->scratch.m0, m0);
    set_vec3s(B(h)->scratch.m1, m1);
}

/// finalize_hydro_forces; out arrays sized by the snapshot count.
/// Each partial row: f[3], f_comp[3], t[3], t_comp[3].
int ref_finalize(void* h, int* n_out, int* ids, double* rows) {
    return guarded([&] {
        RefBlock& b = *B(h);
        const auto parts = psm::finalize_hydro_forces(b.frac, b.scratch, b.box, b.snaps);
        *n_out = static_cast<int>(parts.size());
        for (std::size_t i = 0; i < parts.size(); ++i) {
            ids[i] = parts[i].id;
            const Vec3* v[4] = {&parts[i].f, &parts[i].f_comp, &parts[i].t, &parts[i].t_comp};
            for (int a = 0; a < 4; ++a) {
                rows[12 * i + 3 * a] = v[a]->x;
                rows[12 * i + 3 * a + 1] = v[a]->y;
                rows[12 * i + 3 * a + 2] = v[a]->z;
            }
        }
    });
}

// ------------------------------------------------------------- scenario runs
struct RefSim {
    io::ScenarioConfig cfg;
    std::unique_ptr<Simulation> sim;
};

void* ref_sim_create(const char* json_text) {
    auto* s = new RefSim;
    const int rc = guarded([&] {
        s->cfg = io::parse_config(json_text);
        s->sim = io::build_scenario(s->cfg);
    });
    if (rc != 0) {
        delete s;
        return nullptr;
    }
    return s;
}
void ref_sim_destroy(void* h) { delete static_cast<RefSim*>(h); }

int ref_sim_run(void* h, long steps) {
    return guarded([&] { static_cast<RefSim*>(h)->sim->run(steps); });
}

// Simulation::add_particles with rows {id, x, y, z, r, m} (dropin_sim_add_particles' twin)
int ref_sim_add_particles(void* h, int n, const double* rows) {
    return guarded([&] {
        std::vector<dem::Particle> ps(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            const double* r = rows + 6 * i;
            ps[i].id = static_cast<int>(r[0]);
            ps[i].x = {r[1], r[2], r[3]};
            ps[i].r = r[4];
            ps[i].m = r[5];
        }
        static_cast<RefSim*>(h)->sim->add_particles(ps);
    });
}

void ref_sim_params(void* h, double* tau, double fext[3], int domain[3]) {
    const auto& c = static_cast<RefSim*>(h)->cfg;
    *tau = c.fluid.tau;
    fext[0] = c.fluid.f_ext.x;
    fext[1] = c.fluid.f_ext.y;
    fext[2] = c.fluid.f_ext.z;
    domain[0] = c.domain.x;
    domain[1] = c.domain.y;
    domain[2] = c.domain.z;
}

/// Shear-wave initial state of validation.cpp:46-63 (used by config 2/4).
void ref_sim_shear_wave(void* h) {
    auto& s = *static_cast<RefSim*>(h);
    for (int b = 0; b < s.sim->num_blocks(); ++b) {
        BlockState& blk = s.sim->block(b);
        const Vec3i d = blk.dims();
        // the per-cell arithmetic is independent of the loop order: threads over k planes
        // (a 512^3 domain would otherwise spend ~10 s here before the timed steps)
#pragma omp parallel for schedule(static)
        for (int k = 0; k < d.z; ++k)
            for (int j = 0; j < d.y; ++j)
                for (int i = 0; i < d.x; ++i) {
                    const double gx = blk.box.lo.x + i + 0.5;
                    const double gy = blk.box.lo.y + j + 0.5;
                    const double gz = blk.box.lo.z + k + 0.5;
                    const Vec3 u{0.02 * std::sin(2.0 * dem::kPi * gy / s.cfg.domain.y),
                                 0.015 * std::cos(2.0 * dem::kPi * gz / s.cfg.domain.z),
                                 0.01 * std::sin(2.0 * dem::kPi * gx / s.cfg.domain.x)};
                    const auto feq = lbm::equilibrium(1.0, u);
                    const long base = blk.field.idx(i, j, k);
                    for (int q = 0; q < lbm::kQ; ++q) blk.field.src(q)[base] = feq[q];
                }
    }
}

/// Interior PDFs of the whole domain, global lexicographic (k, j, i), q innermost.
void ref_sim_pdfs(void* h, double* out) {
    auto& s = *static_cast<RefSim*>(h);
    const Vec3i D = s.cfg.domain;
    long n = 0;
    for (int k = 0; k < D.z; ++k)
        for (int j = 0; j < D.y; ++j)
            for (int i = 0; i < D.x; ++i)
                for (int q = 0; q < lbm::kQ; ++q) out[n++] = s.sim->pdf_at({i, j, k}, q);
}

int ref_sim_num_particles(void* h) {
    return static_cast<int>(static_cast<RefSim*>(h)->sim->gather_particles().size());
}

/// Per particle: id, then x u w f_hydro t_hydro (15 doubles) into rows[16*i].
void ref_sim_particles(void* h, double* rows) {
    const auto ps = static_cast<RefSim*>(h)->sim->gather_particles();
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

double ref_sim_mass(void* h) { return static_cast<RefSim*>(h)->sim->total_fluid_mass(); }

/// io::sample_scalars (output.cpp:22-61): step, mass, momentum xyz, fluid KE, particle KE,
/// min gap, max |u|.
int ref_sim_observe(void* h, double out[9]) {
    return guarded([&] {
        const io::ScalarSample s = io::sample_scalars(*static_cast<RefSim*>(h)->sim);
        const double v[9] = {static_cast<double>(s.step), s.mass, s.momentum.x, s.momentum.y,
                             s.momentum.z, s.fluid_ke, s.particle_ke, s.min_gap, s.max_u};
        for (int a = 0; a < 9; ++a) out[a] = v[a];
    });
}

/// io::write_grid_dump (output.cpp:76-107).
int ref_sim_grid_dump(void* h, const char* path) {
    return guarded([&] { io::write_grid_dump(*static_cast<RefSim*>(h)->sim, path); });
}

void ref_sim_reset_timers(void* h) { static_cast<RefSim*>(h)->sim->reset_timers(); }

/// Per-category seconds summed over workers (perf::Category order).
void ref_sim_timings(void* h, double out[8]) {
    const auto per = static_cast<RefSim*>(h)->sim->timings_per_worker();
    for (int c = 0; c < perf::kCategories && c < 8; ++c) {
        out[c] = 0.0;
        for (const auto& t : per) out[c] = std::max(out[c], t.seconds[c]);
    }
}

}  // extern "C"
