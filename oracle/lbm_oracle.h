/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE — plain-C restatement of the reference's GPU-side operators
 * (/root/reference/proj/src/{lbm,psm,boundary,sim}.cpp), used ONLY as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg.
 * Never linked into the product (paper_2303_11811_b200/).
 *
 * Layout conventions are the reference's own:
 *   PDF buffers: 19 q-planes of (nx+2)(ny+2)(nz+2) doubles, plane q at q*alloc,
 *                idx(i,j,k) = ((k+1)(ny+2)+(j+1))(nx+2)+(i+1)      (field.hpp:47-49)
 *   Fraction / velocity / scratch: interior cells, c = (k*ny+j)*nx+i  (field.hpp:95-97)
 *   Vec3 arrays: 3 doubles per cell/particle, xyz interleaved.
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

long orc_alloc_cells(int nx, int ny, int nz);
long orc_idx(int nx, int ny, int i, int j, int k);
void orc_equilibrium(double rho, const double u[3], double feq[19]);

/* lbm.cpp:21-49 — returns the number of unstable cells (NumericError if > 0). */
long orc_collide_stream(int nx, int ny, int nz, const double* src, double* dst, double tau,
                        const double fext[3], const int lo[3], const int hi[3]);
/* lbm.cpp:6-17 */
void orc_stream(int nx, int ny, int nz, const double* src, double* dst, const int lo[3],
                const int hi[3]);

/* psm.cpp:218-262 — fraction arrays are over the block interior. */
long orc_psm_collide_stream(int nx, int ny, int nz, const double* src, double* dst, double tau,
                            const double fext[3], const int lo[3], const int hi[3],
                            const uint8_t* count, const double* b0, const double* b1,
                            const double* btot, const double* v0, const double* v1, double* m0,
                            double* m1);

/* boundary.cpp:98-137 */
void orc_fill_periodic(int nx, int ny, int nz, double* src, const int periodic[3]);
/* boundary.cpp:32-96, 140-146; kinds: 0 periodic, 1 no_slip, 2 velocity, 3 pressure */
void orc_apply_boundaries(int nx, int ny, int nz, double* src, const int kinds[6],
                          const double uwall[18], const double rho[6], const int touches[6]);

/* psm.cpp:12-26 — returns NaN below the validity floor (ConfigError). */
double orc_sphere_volume(double r);
double orc_f_of_r(double r);
/* psm.cpp:28-32 */
double orc_overlap_fraction(const double c[3], const double x[3], double r, double fr);

/* psm.cpp:55-136 (registry + build_fraction_field); returns overfull count. */
long orc_build_fraction_field(const int lo[3], const int dims[3], int n, const int* ids,
                              const double* x, const double* r, const double* fr,
                              int subdivisions, uint8_t* count, int* id0, int* id1, double* b0,
                              double* b1, double* btot);
/* psm.cpp:138-169; returns the unknown-id count (SyncError if > 0). */
long orc_set_solid_velocities(const int lo[3], const int dims[3], int n, const int* ids,
                              const double* x, const double* u, const double* w,
                              const uint8_t* count, const int* id0, const int* id1, double* v0,
                              double* v1);
/* psm.cpp:278-322. rows: n x 12 doubles {f, f_comp, t, t_comp} per snapshot index;
 * used[n] = 1 where the particle got at least one entry. Clears m0/m1 like the
 * reference. Returns 0, or -1 on an unknown id (SyncError). */
int orc_finalize_hydro(const int lo[3], const int dims[3], int n, const int* ids,
                       const double* x, const uint8_t* count, const int* id0, const int* id1,
                       double* m0, double* m1, int* used, double* rows);

/* sim.cpp:120-201 — pack all 19 q of source_slab(off) / unpack into ghost_region(dir). */
long orc_halo_pack(int nx, int ny, int nz, const double* src, const int off[3], double* out);
long orc_halo_unpack(int nx, int ny, int nz, double* src, const int dir[3], const double* in);

uint64_t orc_fnv1a64(const uint8_t* p, long n);

/* lbm.cpp:69-93 (Neumaier-compensated observers) */
double orc_total_mass(int nx, int ny, int nz, const double* src);
void orc_total_momentum(int nx, int ny, int nz, const double* src, double out[3]);

#ifdef __cplusplus
}
#endif
#endif
