/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — plain-C restatement of the reference's GPU-side operators.
 * It is the parity CHECKER for the CUDA path, never the thing measured or shipped.
 * Each function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). The arithmetic keeps the reference's operation order
 * term by term (C++ left-to-right evaluation, -ffp-contract=off), so results
 * agree bitwise with the reference built with its own flags (CMakeLists.txt:12-14).
 * Pinned against oracle/_ref (the reference itself) in tests/test_oracle.py.
 */
#include "lbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* lattice.hpp:18-29 — rest, then opposite pairs. */
static const int C[19][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                             {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                             {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                             {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
/* lattice.hpp:32-39 — numerators over 36, rounded once. */
static const int WNUM[19] = {12, 2, 2, 2, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
static double W(int q) { return WNUM[q] / 36.0; }
static int opposite(int q) { return q == 0 ? 0 : (((q - 1) ^ 1) + 1); } /* lattice.hpp:46 */

static const double kRho0 = 1.0, kDt = 1.0, kInvCs2 = 3.0, kInvCs4 = 9.0; /* lbm.hpp:15-16, lattice.hpp:41-43 */
static const double kMaxVelocity = 0.57;                                  /* lbm.hpp:19 */

long orc_alloc_cells(int nx, int ny, int nz) { return (long)(nx + 2) * (ny + 2) * (nz + 2); }

/* field.hpp:47-49 */
long orc_idx(int nx, int ny, int i, int j, int k) {
    return ((long)(k + 1) * (ny + 2) + (j + 1)) * (nx + 2) + (i + 1);
}

/* field.hpp:51-54 */
static long shift(int nx, int ny, int q) {
    return C[q][0] + (long)C[q][1] * (nx + 2) + (long)C[q][2] * (nx + 2) * (ny + 2);
}

static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

/* lbm.hpp:38-45 */
void orc_equilibrium(double rho, const double u[3], double feq[19]) {
    const double u_sq = dot3(u, u);
    for (int q = 0; q < 19; ++q) {
        const double c[3] = {C[q][0], C[q][1], C[q][2]};
        const double cu = dot3(c, u);
        feq[q] = W(q) * (rho + kRho0 * (cu * kInvCs2 + 0.5 * cu * cu * kInvCs4 - 0.5 * u_sq * kInvCs2));
    }
}

/* lbm.hpp:93-124 — collide_cell */
static int collide_cell(double f[19], const double fext[3], double inv_tau) {
    double rho = 0.0, ux = 0.0, uy = 0.0, uz = 0.0;
    for (int q = 0; q < 19; ++q) {
        rho += f[q];
        ux += f[q] * C[q][0];
        uy += f[q] * C[q][1];
        uz += f[q] * C[q][2];
    }
    ux /= kRho0;
    uy /= kRho0;
    uz /= kRho0;
    const double u_sq = ux * ux + uy * uy + uz * uz;
    const int ok = rho > 0.0 && u_sq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    const int forced = fext[0] != 0.0 || fext[1] != 0.0 || fext[2] != 0.0;
    for (int q = 0; q < 19; ++q) {
        const double cx = C[q][0], cy = C[q][1], cz = C[q][2];
        const double cu = cx * ux + cy * uy + cz * uz;
        const double feq = W(q) * (rho + kRho0 * (cu * kInvCs2 + 0.5 * cu * cu * kInvCs4 - 0.5 * u_sq * kInvCs2));
        double out = f[q] + inv_tau * (feq - f[q]);
        if (forced) {
            const double bx = (cx - ux) * kInvCs2 + cu * kInvCs4 * cx;
            const double by = (cy - uy) * kInvCs2 + cu * kInvCs4 * cy;
            const double bz = (cz - uz) * kInvCs2 + cu * kInvCs4 * cz;
            out += kDt * W(q) * (bx * fext[0] + by * fext[1] + bz * fext[2]);
        }
        f[q] = out;
    }
    return ok;
}

/* lbm.cpp:21-49 — collide_stream_impl (pull, collide, store) */
long orc_collide_stream(int nx, int ny, int nz, const double* src, double* dst, double tau,
                        const double fext[3], const int lo[3], const int hi[3]) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const double inv_tau = kDt / tau;
    long bad = 0;
    for (int k = lo[2]; k < hi[2]; ++k)
        for (int j = lo[1]; j < hi[1]; ++j) {
            long base = orc_idx(nx, ny, lo[0], j, k);
            for (int i = lo[0]; i < hi[0]; ++i, ++base) {
                double f[19];
                for (int q = 0; q < 19; ++q) f[q] = src[q * alloc + base - shift(nx, ny, q)];
                if (!collide_cell(f, fext, inv_tau)) ++bad;
                for (int q = 0; q < 19; ++q) dst[q * alloc + base] = f[q];
            }
        }
    return bad;
}

/* lbm.cpp:6-17 */
void orc_stream(int nx, int ny, int nz, const double* src, double* dst, const int lo[3],
                const int hi[3]) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    for (int q = 0; q < 19; ++q) {
        const long sh = shift(nx, ny, q);
        for (int k = lo[2]; k < hi[2]; ++k)
            for (int j = lo[1]; j < hi[1]; ++j) {
                long base = orc_idx(nx, ny, lo[0], j, k);
                for (int i = lo[0]; i < hi[0]; ++i, ++base)
                    dst[q * alloc + base] = src[q * alloc + base - sh];
            }
    }
}

/* psm.cpp:174-216 — psm_cell */
static int psm_cell(double f[19], const double fext[3], double inv_tau, int cnt, double b_tot,
                    const double b_entry[2], const double u_entry[2][3], double m_out[2][3]) {
    double rho = 0.0, mom[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < 19; ++q) {
        rho += f[q];
        mom[0] += f[q] * C[q][0];
        mom[1] += f[q] * C[q][1];
        mom[2] += f[q] * C[q][2];
    }
    const double u[3] = {mom[0] / kRho0, mom[1] / kRho0, mom[2] / kRho0};
    const double u_sq = dot3(u, u);
    const int ok = rho > 0.0 && u_sq <= kMaxVelocity * kMaxVelocity && isfinite(rho);

    double feq_f[19];
    orc_equilibrium(rho, u, feq_f);

    double fout[19];
    const double fluid_w = 1.0 - b_tot;
    for (int q = 0; q < 19; ++q) {
        const double c[3] = {C[q][0], C[q][1], C[q][2]};
        const double cu = dot3(c, u);
        double bracket[3];
        for (int a = 0; a < 3; ++a) bracket[a] = (c[a] - u[a]) * kInvCs2 + (cu * kInvCs4) * c[a];
        const double fq_force = kDt * W(q) * dot3(bracket, fext);
        fout[q] = f[q] + fluid_w * (inv_tau * (feq_f[q] - f[q]) + fq_force);
    }

    for (int e = 0; e < cnt; ++e) {
        double feq_p[19];
        orc_equilibrium(rho, u_entry[e], feq_p);
        double m[3] = {0.0, 0.0, 0.0};
        for (int q = 0; q < 19; ++q) {
            const int qb = opposite(q);
            const double c_solid = (f[qb] - feq_f[qb]) - (f[q] - feq_p[q]);
            fout[q] += b_entry[e] * c_solid;
            m[0] -= c_solid * (double)C[q][0];
            m[1] -= c_solid * (double)C[q][1];
            m[2] -= c_solid * (double)C[q][2];
        }
        for (int a = 0; a < 3; ++a) m_out[e][a] = b_entry[e] * m[a];
    }
    memcpy(f, fout, sizeof(fout));
    return ok;
}

/* psm.cpp:218-262 — psm_collide_stream_impl */
long orc_psm_collide_stream(int nx, int ny, int nz, const double* src, double* dst, double tau,
                            const double fext[3], const int lo[3], const int hi[3],
                            const uint8_t* count, const double* b0, const double* b1,
                            const double* btot, const double* v0, const double* v1, double* m0,
                            double* m1) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const double inv_tau = kDt / tau;
    long bad = 0;
    for (int k = lo[2]; k < hi[2]; ++k)
        for (int j = lo[1]; j < hi[1]; ++j) {
            long base = orc_idx(nx, ny, lo[0], j, k);
            long fc = ((long)k * ny + j) * nx + lo[0];
            for (int i = lo[0]; i < hi[0]; ++i, ++base, ++fc) {
                double f[19];
                for (int q = 0; q < 19; ++q) f[q] = src[q * alloc + base - shift(nx, ny, q)];
                const int cnt = count[fc];
                if (cnt == 0) {
                    if (!collide_cell(f, fext, inv_tau)) ++bad;
                } else {
                    const double be[2] = {b0[fc], b1[fc]};
                    double ue[2][3], m[2][3];
                    for (int a = 0; a < 3; ++a) {
                        ue[0][a] = v0[3 * fc + a];
                        ue[1][a] = v1[3 * fc + a];
                    }
                    if (!psm_cell(f, fext, inv_tau, cnt, btot[fc], be, ue, m)) ++bad;
                    for (int a = 0; a < 3; ++a) m0[3 * fc + a] = m[0][a];
                    if (cnt > 1)
                        for (int a = 0; a < 3; ++a) m1[3 * fc + a] = m[1][a];
                }
                for (int q = 0; q < 19; ++q) dst[q * alloc + base] = f[q];
            }
        }
    return bad;
}

/* boundary.cpp:98-137 — fill_periodic_ghosts */
void orc_fill_periodic(int nx, int ny, int nz, double* src, const int periodic[3]) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const int dims[3] = {nx, ny, nz};
    for (int ox = -1; ox <= 1; ++ox)
        for (int oy = -1; oy <= 1; ++oy)
            for (int oz = -1; oz <= 1; ++oz) {
                const int off[3] = {ox, oy, oz};
                if (ox == 0 && oy == 0 && oz == 0) continue;
                int ok = 1;
                for (int a = 0; a < 3; ++a)
                    if (off[a] != 0 && !periodic[a]) ok = 0;
                if (!ok) continue;
                int lo[3], hi[3];
                for (int a = 0; a < 3; ++a) {
                    if (off[a] == -1) {
                        lo[a] = -1;
                        hi[a] = 0;
                    } else if (off[a] == 1) {
                        lo[a] = dims[a];
                        hi[a] = dims[a] + 1;
                    } else {
                        lo[a] = 0;
                        hi[a] = dims[a];
                    }
                }
                for (int q = 0; q < 19; ++q) {
                    double* p = src + q * alloc;
                    for (int k = lo[2]; k < hi[2]; ++k)
                        for (int j = lo[1]; j < hi[1]; ++j)
                            for (int i = lo[0]; i < hi[0]; ++i) {
                                const int si = ox == 0 ? i : (ox == 1 ? 0 : nx - 1);
                                const int sj = oy == 0 ? j : (oy == 1 ? 0 : ny - 1);
                                const int sk = oz == 0 ? k : (oz == 1 ? 0 : nz - 1);
                                p[orc_idx(nx, ny, i, j, k)] = p[orc_idx(nx, ny, si, sj, sk)];
                            }
                }
            }
}

/* boundary.cpp:75-80 — cell_velocity (bare first moment) */
static void cell_velocity(int nx, int ny, int nz, const double* src, const int s[3], double u[3]) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const long base = orc_idx(nx, ny, s[0], s[1], s[2]);
    double mom[3] = {0.0, 0.0, 0.0};
    for (int q = 0; q < 19; ++q) {
        const double v = src[q * alloc + base];
        mom[0] += v * (double)C[q][0];
        mom[1] += v * (double)C[q][1];
        mom[2] += v * (double)C[q][2];
    }
    for (int a = 0; a < 3; ++a) u[a] = mom[a] / kRho0;
}

/* boundary.cpp:82-136 — fill_face */
static void fill_face(int nx, int ny, int nz, double* src, const int kinds[6],
                      const double uwall[18], const double rho[6], const int touches[6], int face) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const int dims[3] = {nx, ny, nz};
    const int axis = face / 2, side = face % 2;
    const int kind = kinds[face];
    const int ga = side == 0 ? -1 : dims[axis];
    const int b = (axis + 1) % 3, c = (axis + 2) % 3;
    for (int jb = -1; jb <= dims[b]; ++jb)
        for (int jc = -1; jc <= dims[c]; ++jc) {
            int g[3];
            g[axis] = ga;
            g[b] = jb;
            g[c] = jc;
            for (int q = 1; q < 19; ++q) {
                const int s[3] = {g[0] + C[q][0], g[1] + C[q][1], g[2] + C[q][2]};
                if (!(s[0] >= 0 && s[0] < nx && s[1] >= 0 && s[1] < ny && s[2] >= 0 && s[2] < nz))
                    continue;
                int multi_wall = 0;
                for (int a2 = 0; a2 < 3; ++a2) {
                    if (a2 == axis) continue;
                    if (g[a2] == -1 && touches[2 * a2] && kinds[2 * a2] != 0) multi_wall = 1;
                    if (g[a2] == dims[a2] && touches[2 * a2 + 1] && kinds[2 * a2 + 1] != 0)
                        multi_wall = 1;
                }
                const int qb = opposite(q);
                const long gi = orc_idx(nx, ny, g[0], g[1], g[2]);
                const long si = orc_idx(nx, ny, s[0], s[1], s[2]);
                const double out = src[qb * alloc + si];
                const double cq[3] = {C[q][0], C[q][1], C[q][2]};
                double v;
                if (multi_wall || kind == 1) {
                    v = out;
                } else if (kind == 2) {
                    v = out + 2.0 * W(q) * kRho0 * dot3(cq, &uwall[3 * face]) * kInvCs2;
                } else {
                    double ub[3];
                    cell_velocity(nx, ny, nz, src, s, ub);
                    const double cu = dot3(cq, ub);
                    const double feq_even =
                        W(q) * (rho[face] + kRho0 * (0.5 * cu * cu * kInvCs4 - 0.5 * dot3(ub, ub) * kInvCs2));
                    v = -out + 2.0 * feq_even;
                }
                src[q * alloc + gi] = v;
            }
        }
}

/* boundary.cpp:140-146 */
void orc_apply_boundaries(int nx, int ny, int nz, double* src, const int kinds[6],
                          const double uwall[18], const double rho[6], const int touches[6]) {
    for (int face = 0; face < 6; ++face) {
        if (!touches[face]) continue;
        if (kinds[face] == 0) continue;
        fill_face(nx, ny, nz, src, kinds, uwall, rho, touches, face);
    }
}

/* psm.cpp:12-18 */
double orc_sphere_volume(double r) {
    const double r2 = r * r;
    const double s = sqrt(r2 - 0.5);
    return (1.0 / 12.0 - r2) * atan(0.5 * s / (0.5 - r2)) + s / 3.0 +
           (r2 - 1.0 / 12.0) * atan(0.5 / s) - (4.0 / 3.0) * r2 * r * atan(0.25 / (r * s));
}

/* psm.cpp:20-26 */
double orc_f_of_r(double r) {
    const double floor_r = sqrt(0.5);
    if (!(r >= floor_r)) return NAN;
    return orc_sphere_volume(r) - r + 0.5;
}

/* psm.cpp:28-32, with std::clamp(v, lo, hi) = v < lo ? lo : (hi < v ? hi : v) */
double orc_overlap_fraction(const double c[3], const double x[3], double r, double fr) {
    const double d[3] = {c[0] - x[0], c[1] - x[1], c[2] - x[2]};
    const double dist = sqrt(dot3(d, d));
    const double eps = -(dist - r) + fr;
    return eps < 0.0 ? 0.0 : (1.0 < eps ? 1.0 : eps);
}

/* psm.cpp:37-44 */
static double dist2_point_box(const double p[3], const double lo[3], const double hi[3]) {
    double d2 = 0.0;
    for (int a = 0; a < 3; ++a) {
        const double v = p[a] < lo[a] ? lo[a] - p[a] : (p[a] > hi[a] ? p[a] - hi[a] : 0.0);
        d2 += v * v;
    }
    return d2;
}

/* psm.cpp:55-85 (SubBlockRegistry::build) + 93-136 (build_fraction_field) */
long orc_build_fraction_field(const int lo[3], const int dims[3], int n, const int* ids,
                              const double* x, const double* r, const double* fr,
                              int subdivisions, uint8_t* count, int* id0, int* id1, double* b0,
                              double* b1, double* btot) {
    const int K = subdivisions;
    int ext[3];
    for (int a = 0; a < 3; ++a) {
        ext[a] = (dims[a] + K - 1) / K;
        if (ext[a] < 1) ext[a] = 1;
    }
    const long nsub = (long)K * K * K;
    int* len = calloc(nsub, sizeof(int));
    int** lists = calloc(nsub, sizeof(int*));
    for (int p = 0; p < n; ++p) {
        const double reach = r[p] + 0.5;
        for (int sk = 0; sk < K; ++sk)
            for (int sj = 0; sj < K; ++sj)
                for (int si = 0; si < K; ++si) {
                    const double blo[3] = {(double)(lo[0] + si * ext[0]), (double)(lo[1] + sj * ext[1]),
                                           (double)(lo[2] + sk * ext[2])};
                    double bhi[3];
                    for (int a = 0; a < 3; ++a) {
                        const double e = blo[a] + ext[a], h = (double)(lo[a] + dims[a]);
                        bhi[a] = h < e ? h : e; /* std::min<double>(lo+ext, box.hi) */
                    }
                    if (bhi[0] <= blo[0] || bhi[1] <= blo[1] || bhi[2] <= blo[2]) continue;
                    if (dist2_point_box(&x[3 * p], blo, bhi) <= reach * reach) {
                        const long s = ((long)sk * K + sj) * K + si;
                        lists[s] = realloc(lists[s], (len[s] + 1) * sizeof(int));
                        lists[s][len[s]++] = p;
                    }
                }
    }
    long overfull = 0;
    for (int k = 0; k < dims[2]; ++k)
        for (int j = 0; j < dims[1]; ++j)
            for (int i = 0; i < dims[0]; ++i) {
                const long c = ((long)k * dims[1] + j) * dims[0] + i;
                const double center[3] = {(double)(lo[0] + i) + 0.5, (double)(lo[1] + j) + 0.5,
                                          (double)(lo[2] + k) + 0.5};
                const long s = ((long)(k / ext[2]) * K + (j / ext[1])) * K + (i / ext[0]);
                int cnt = 0;
                double sum = 0.0;
                for (int t = 0; t < len[s]; ++t) {
                    const int p = lists[s][t];
                    const double eps = orc_overlap_fraction(center, &x[3 * p], r[p], fr[p]);
                    if (eps <= 0.0) continue;
                    if (cnt == 0) {
                        id0[c] = ids[p];
                        b0[c] = eps;
                    } else if (cnt == 1) {
                        id1[c] = ids[p];
                        b1[c] = eps;
                    } else {
                        ++overfull;
                        break;
                    }
                    ++cnt;
                    sum += eps;
                }
                count[c] = (uint8_t)cnt;
                btot[c] = sum < 1.0 ? sum : 1.0; /* std::min(1.0, sum) */
            }
    for (long s = 0; s < nsub; ++s) free(lists[s]);
    free(lists);
    free(len);
    return overfull;
}

/* psm.cpp:46-51 */
static int snapshot_index(int n, const int* ids, int id) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (ids[mid] < id)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < n && ids[lo] == id) ? lo : -1;
}

/* vec3.hpp:92-94 */
static void cross3(const double a[3], const double b[3], double out[3]) {
    out[0] = a[1] * b[2] - a[2] * b[1];
    out[1] = a[2] * b[0] - a[0] * b[2];
    out[2] = a[0] * b[1] - a[1] * b[0];
}

/* psm.cpp:138-169 */
long orc_set_solid_velocities(const int lo[3], const int dims[3], int n, const int* ids,
                              const double* x, const double* u, const double* w,
                              const uint8_t* count, const int* id0, const int* id1, double* v0,
                              double* v1) {
    long unknown = 0;
    for (int k = 0; k < dims[2]; ++k)
        for (int j = 0; j < dims[1]; ++j)
            for (int i = 0; i < dims[0]; ++i) {
                const long c = ((long)k * dims[1] + j) * dims[0] + i;
                const int cnt = count[c];
                if (cnt == 0) continue;
                const double center[3] = {(double)(lo[0] + i) + 0.5, (double)(lo[1] + j) + 0.5,
                                          (double)(lo[2] + k) + 0.5};
                for (int e = 0; e < cnt; ++e) {
                    const int id = e == 0 ? id0[c] : id1[c];
                    const int p = snapshot_index(n, ids, id);
                    if (p < 0) {
                        ++unknown;
                        continue;
                    }
                    const double rr[3] = {center[0] - x[3 * p], center[1] - x[3 * p + 1],
                                          center[2] - x[3 * p + 2]};
                    double cr[3];
                    cross3(&w[3 * p], rr, cr);
                    double* v = (e == 0 ? v0 : v1) + 3 * c;
                    for (int a = 0; a < 3; ++a) v[a] = u[3 * p + a] + cr[a];
                }
            }
    return unknown;
}

/* vec3.hpp:75-82 — Neumaier add */
static void comp_add(double* sum, double* comp, double v) {
    const double t = *sum + v;
    if (fabs(*sum) >= fabs(v))
        *comp += (*sum - t) + v;
    else
        *comp += (v - t) + *sum;
    *sum = t;
}

/* psm.cpp:278-322 */
int orc_finalize_hydro(const int lo[3], const int dims[3], int n, const int* ids,
                       const double* x, const uint8_t* count, const int* id0, const int* id1,
                       double* m0, double* m1, int* used, double* rows) {
    memset(used, 0, sizeof(int) * (size_t)n);
    memset(rows, 0, sizeof(double) * 12 * (size_t)n);
    for (int k = 0; k < dims[2]; ++k)
        for (int j = 0; j < dims[1]; ++j)
            for (int i = 0; i < dims[0]; ++i) {
                const long c = ((long)k * dims[1] + j) * dims[0] + i;
                const int cnt = count[c];
                if (cnt == 0) continue;
                const double center[3] = {(double)(lo[0] + i) + 0.5, (double)(lo[1] + j) + 0.5,
                                          (double)(lo[2] + k) + 0.5};
                for (int e = 0; e < cnt; ++e) {
                    const int id = e == 0 ? id0[c] : id1[c];
                    const int p = snapshot_index(n, ids, id);
                    if (p < 0) return -1;
                    double* m = (e == 0 ? m0 : m1) + 3 * c;
                    double* row = rows + 12 * p;
                    for (int a = 0; a < 3; ++a) comp_add(&row[a], &row[3 + a], m[a]);
                    const double rr[3] = {center[0] - x[3 * p], center[1] - x[3 * p + 1],
                                          center[2] - x[3 * p + 2]};
                    double tq[3];
                    cross3(rr, m, tq);
                    for (int a = 0; a < 3; ++a) comp_add(&row[6 + a], &row[9 + a], tq[a]);
                    used[p] = 1;
                    m[0] = m[1] = m[2] = 0.0;
                }
            }
    return 0;
}

/* sim.cpp:120-135 (source_slab) and 156-179 (pack loop, q-major then k, j, i) */
long orc_halo_pack(int nx, int ny, int nz, const double* src, const int off[3], double* out) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const int dims[3] = {nx, ny, nz};
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        if (off[a] == 1) {
            lo[a] = dims[a] - 1;
            hi[a] = dims[a];
        } else if (off[a] == -1) {
            lo[a] = 0;
            hi[a] = 1;
        } else {
            lo[a] = 0;
            hi[a] = dims[a];
        }
    }
    long v = 0;
    for (int q = 0; q < 19; ++q)
        for (int k = lo[2]; k < hi[2]; ++k)
            for (int j = lo[1]; j < hi[1]; ++j)
                for (int i = lo[0]; i < hi[0]; ++i) out[v++] = src[q * alloc + orc_idx(nx, ny, i, j, k)];
    return v;
}

/* sim.cpp:137-152 (ghost_region) and 181-201 (unpack loop) */
long orc_halo_unpack(int nx, int ny, int nz, double* src, const int dir[3], const double* in) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    const int dims[3] = {nx, ny, nz};
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        if (dir[a] == 1) {
            lo[a] = dims[a];
            hi[a] = dims[a] + 1;
        } else if (dir[a] == -1) {
            lo[a] = -1;
            hi[a] = 0;
        } else {
            lo[a] = 0;
            hi[a] = dims[a];
        }
    }
    long v = 0;
    for (int q = 0; q < 19; ++q)
        for (int k = lo[2]; k < hi[2]; ++k)
            for (int j = lo[1]; j < hi[1]; ++j)
                for (int i = lo[0]; i < hi[0]; ++i) src[q * alloc + orc_idx(nx, ny, i, j, k)] = in[v++];
    return v;
}

/* lbm.cpp:69-80 */
double orc_total_mass(int nx, int ny, int nz, const double* src) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    double sum = 0.0, comp = 0.0;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const long base = orc_idx(nx, ny, i, j, k);
                double rho = 0.0;
                for (int q = 0; q < 19; ++q) rho += src[q * alloc + base];
                comp_add(&sum, &comp, rho);
            }
    return sum + comp;
}

/* lbm.cpp:82-93 */
void orc_total_momentum(int nx, int ny, int nz, const double* src, double out[3]) {
    const long alloc = orc_alloc_cells(nx, ny, nz);
    double sum[3] = {0, 0, 0}, comp[3] = {0, 0, 0};
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const long base = orc_idx(nx, ny, i, j, k);
                double m[3] = {0.0, 0.0, 0.0};
                for (int q = 0; q < 19; ++q) {
                    const double v = src[q * alloc + base];
                    m[0] += v * (double)C[q][0];
                    m[1] += v * (double)C[q][1];
                    m[2] += v * (double)C[q][2];
                }
                for (int a = 0; a < 3; ++a) comp_add(&sum[a], &comp[a], m[a]);
            }
    for (int a = 0; a < 3; ++a) out[a] = sum[a] + comp[a];
}

/* FNV-1a 64 over raw bytes — the run-report hash of config.cpp:294-302, used on the PDF
 * dump (k, j, i, q order) as the known-answer fingerprint of SURVEY.md §8(c). */
uint64_t orc_fnv1a64(const uint8_t* p, long n) {
    uint64_t h = 1469598103934665603ull;
    for (long i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}
