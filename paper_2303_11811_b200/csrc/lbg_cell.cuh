// SPDX-License-Identifier: Apache-2.0
//
// Per-cell D3Q19 operators, bit-compatible with the reference C++ (built with
// -ffp-contract=off): this code is compiled with --fmad=false and keeps every
// nonzero term in the reference's left-to-right order.
//
// srt_cell: collide_cell (lbm.hpp:93-124). The zero-velocity terms of the reference
// sums (f * 0.0) are dropped by hand: adding a signed zero to a nonzero partial sum is
// exact, and the opposite-direction pair shares |cu| exactly (IEEE rounding is
// symmetric under negation), so each pair costs one cu, one cu*3 and one cu^2 term.
// psm_cell: the covered-cell operator (psm.cpp:174-216), written term by term.
#pragma once

#include "lbg_internal.cuh"

namespace lbg {

// equilibrium numerator pair for +cu / -cu: feq = w (rho + ((+-A + B) - T))  (lbm.hpp:38-45)
__device__ __forceinline__ void feq_pair(double w, double cu, double rho, double T, double& fp,
                                         double& fm) {
    const double A = cu * 3.0;
    const double B = ((0.5 * cu) * cu) * 9.0;
    fp = w * (rho + ((A + B) - T));
    fm = w * (rho + ((B - A) - T));
}

// Guo-style forcing of lbm.hpp:115-120 for direction q (generic: exact by construction).
template <int q>
__device__ __forceinline__ double forcing(double cu, double ux, double uy, double uz, double fx,
                                          double fy, double fz) {
    constexpr double c0 = cx(q), c1 = cy(q), c2 = cz(q);
    const double bx = (c0 - ux) * 3.0 + (cu * 9.0) * c0;
    const double by = (c1 - uy) * 3.0 + (cu * 9.0) * c1;
    const double bz = (c2 - uz) * 3.0 + (cu * 9.0) * c2;
    return (1.0 * wq(q)) * ((bx * fx + by * fy) + bz * fz);
}

struct Force {
    double x, y, z;
};

// collide_cell (lbm.hpp:93-124): f in/out, returns the stability predicate.
template <bool kForced>
__device__ __forceinline__ bool srt_cell(double (&f)[kQ], double inv_tau, Force F) {
    double rho = f[0];
#pragma unroll
    for (int q = 1; q < kQ; ++q) rho += f[q];
    const double ux = ((((((((f[1] - f[2]) + f[7]) - f[8]) + f[9]) - f[10]) + f[11]) - f[12]) + f[13]) - f[14];
    const double uy = ((((((((f[3] - f[4]) + f[7]) - f[8]) - f[9]) + f[10]) + f[15]) - f[16]) + f[17]) - f[18];
    const double uz = ((((((((f[5] - f[6]) + f[11]) - f[12]) - f[13]) + f[14]) + f[15]) - f[16]) - f[17]) + f[18];
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const bool ok = rho > 0.0 && usq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    const double T = (0.5 * usq) * 3.0;

    // cu per direction; opposite directions are exact negations
    const double cu[kQ] = {0.0,       ux,        -ux,       uy,        -uy,       uz,        -uz,
                           ux + uy,   -(ux + uy), ux - uy,  -(ux - uy), ux + uz,  -(ux + uz),
                           ux - uz,   -(ux - uz), uy + uz,  -(uy + uz), uy - uz,  -(uy - uz)};
    double feq[kQ];
    feq[0] = wq(0) * (rho - T);  // cu = 0: rho + ((+0) - T)
    feq_pair(wq(1), ux, rho, T, feq[1], feq[2]);
    feq_pair(wq(3), uy, rho, T, feq[3], feq[4]);
    feq_pair(wq(5), uz, rho, T, feq[5], feq[6]);
    feq_pair(wq(7), cu[7], rho, T, feq[7], feq[8]);
    feq_pair(wq(9), cu[9], rho, T, feq[9], feq[10]);
    feq_pair(wq(11), cu[11], rho, T, feq[11], feq[12]);
    feq_pair(wq(13), cu[13], rho, T, feq[13], feq[14]);
    feq_pair(wq(15), cu[15], rho, T, feq[15], feq[16]);
    feq_pair(wq(17), cu[17], rho, T, feq[17], feq[18]);

#pragma unroll
    for (int q = 0; q < kQ; ++q) f[q] = f[q] + inv_tau * (feq[q] - f[q]);

    if constexpr (kForced) {
#define LBG_F(q) f[q] += forcing<q>(cu[q], ux, uy, uz, F.x, F.y, F.z)
        LBG_F(0); LBG_F(1); LBG_F(2); LBG_F(3); LBG_F(4); LBG_F(5); LBG_F(6);
        LBG_F(7); LBG_F(8); LBG_F(9); LBG_F(10); LBG_F(11); LBG_F(12);
        LBG_F(13); LBG_F(14); LBG_F(15); LBG_F(16); LBG_F(17); LBG_F(18);
#undef LBG_F
    }
    return ok;
}

// equilibrium() term by term (lbm.hpp:38-45), generic velocity.
__device__ __forceinline__ void equilibrium(double rho, double u0, double u1, double u2,
                                            double (&feq)[kQ]) {
    const double u_sq = (u0 * u0 + u1 * u1) + u2 * u2;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double c0 = cx(q), c1 = cy(q), c2 = cz(q);
        const double cu = (c0 * u0 + c1 * u1) + c2 * u2;
        feq[q] = wq(q) * (rho + 1.0 * (((cu * 3.0) + ((0.5 * cu) * cu) * 9.0) - (0.5 * u_sq) * 3.0));
    }
}

// psm_cell (psm.cpp:174-216). m_out[e] = B_e * sum_q C_solid,q * c_qbar.
__device__ __forceinline__ bool psm_cell(double (&f)[kQ], double inv_tau, Force F, int cnt,
                                         double b_tot, const double be[2], const double ue[2][3],
                                         double m_out[2][3]) {
    double rho = 0.0, m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        rho += f[q];
        m0 += (double)cx(q) * f[q];
        m1 += (double)cy(q) * f[q];
        m2 += (double)cz(q) * f[q];
    }
    const double u0 = m0 / 1.0, u1 = m1 / 1.0, u2 = m2 / 1.0;
    const double u_sq = (u0 * u0 + u1 * u1) + u2 * u2;
    const bool ok = rho > 0.0 && u_sq <= kMaxVelocity * kMaxVelocity && isfinite(rho);

    double feq_f[kQ];
    equilibrium(rho, u0, u1, u2, feq_f);
    double fout[kQ];
    const double fluid_w = 1.0 - b_tot;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double c0 = cx(q), c1 = cy(q), c2 = cz(q);
        const double cu = (c0 * u0 + c1 * u1) + c2 * u2;
        const double bx = (c0 - u0) * 3.0 + (cu * 9.0) * c0;
        const double by = (c1 - u1) * 3.0 + (cu * 9.0) * c1;
        const double bz = (c2 - u2) * 3.0 + (cu * 9.0) * c2;
        const double fq_force = (1.0 * wq(q)) * ((bx * F.x + by * F.y) + bz * F.z);
        fout[q] = f[q] + fluid_w * (inv_tau * (feq_f[q] - f[q]) + fq_force);
    }
    for (int e = 0; e < cnt; ++e) {
        double feq_p[kQ];
        equilibrium(rho, ue[e][0], ue[e][1], ue[e][2], feq_p);
        double mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const int qb = opposite(q);
            const double c_solid = (f[qb] - feq_f[qb]) - (f[q] - feq_p[q]);
            fout[q] += be[e] * c_solid;
            // c_q = 0 terms subtract a signed zero from a sum that starts at +0 and
            // can never become -0 (x - x is +0), so they are skipped exactly
            if (cx(q) != 0) mx -= c_solid * (double)cx(q);
            if (cy(q) != 0) my -= c_solid * (double)cy(q);
            if (cz(q) != 0) mz -= c_solid * (double)cz(q);
        }
        m_out[e][0] = be[e] * mx;
        m_out[e][1] = be[e] * my;
        m_out[e][2] = be[e] * mz;
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) f[q] = fout[q];
    return ok;
}

// moments of srt_cell (folded, identical operations)
__device__ __forceinline__ void moments(const double (&f)[kQ], double& rho, double& ux, double& uy,
                                        double& uz) {
    rho = f[0];
#pragma unroll
    for (int q = 1; q < kQ; ++q) rho += f[q];
    ux = ((((((((f[1] - f[2]) + f[7]) - f[8]) + f[9]) - f[10]) + f[11]) - f[12]) + f[13]) - f[14];
    uy = ((((((((f[3] - f[4]) + f[7]) - f[8]) - f[9]) + f[10]) + f[15]) - f[16]) + f[17]) - f[18];
    uz = ((((((((f[5] - f[6]) + f[11]) - f[12]) - f[13]) + f[14]) + f[15]) - f[16]) - f[17]) + f[18];
}

// equilibrium(rho, u) via the exact +-cu pairs (any velocity; signed zeros in cu cannot
// reach feq because A + B and B - A with B = +0 are +0 either way)
__device__ __forceinline__ void feq_all(double rho, double ux, double uy, double uz, double (&feq)[kQ]) {
    const double T = (0.5 * ((ux * ux + uy * uy) + uz * uz)) * 3.0;
    feq[0] = wq(0) * (rho - T);
    feq_pair(wq(1), ux, rho, T, feq[1], feq[2]);
    feq_pair(wq(3), uy, rho, T, feq[3], feq[4]);
    feq_pair(wq(5), uz, rho, T, feq[5], feq[6]);
    feq_pair(wq(7), ux + uy, rho, T, feq[7], feq[8]);
    feq_pair(wq(9), ux - uy, rho, T, feq[9], feq[10]);
    feq_pair(wq(11), ux + uz, rho, T, feq[11], feq[12]);
    feq_pair(wq(13), ux - uz, rho, T, feq[13], feq[14]);
    feq_pair(wq(15), uy + uz, rho, T, feq[15], feq[16]);
    feq_pair(wq(17), uy - uz, rho, T, feq[17], feq[18]);
}

// cu of direction q for velocity u, equal to (c . u) of the reference for nonzero results
template <int q>
__device__ __forceinline__ double cu_of(double ux, double uy, double uz) {
    constexpr int a = cx(q), b = cy(q), c = cz(q);
    if constexpr (a == 0 && b == 0 && c == 0) return 0.0;
    else if constexpr (b == 0 && c == 0) return a > 0 ? ux : -ux;
    else if constexpr (a == 0 && c == 0) return b > 0 ? uy : -uy;
    else if constexpr (a == 0 && b == 0) return c > 0 ? uz : -uz;
    else if constexpr (c == 0) return a > 0 ? (b > 0 ? ux + uy : ux - uy) : (b > 0 ? -(ux - uy) : -(ux + uy));
    else if constexpr (b == 0) return a > 0 ? (c > 0 ? ux + uz : ux - uz) : (c > 0 ? -(ux - uz) : -(ux + uz));
    else return b > 0 ? (c > 0 ? uy + uz : uy - uz) : (c > 0 ? -(uy - uz) : -(uy + uz));
}

// psm_cell (psm.cpp:174-216) with the register footprint cut down: the fluid equilibrium
// enters only through d_q = f_q - feq_f,q (feq_f - f == -d exactly), the particle
// equilibria are rebuilt pairwise per entry, and the unforced path drops the force term
// (it adds a signed zero to a value it cannot change). Momentum sums keep every term.
template <bool kForced>
__device__ __forceinline__ bool psm_cell_opt(double (&f)[kQ], double inv_tau, Force F, int cnt,
                                             double b_tot, const double be[2], const double ue[2][3],
                                             double m_out[2][3]) {
    double rho, ux, uy, uz;
    moments(f, rho, ux, uy, uz);
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const bool ok = rho > 0.0 && usq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    double d[kQ];
    feq_all(rho, ux, uy, uz, d);
    double fout[kQ];
    const double fluid_w = 1.0 - b_tot;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double coll = inv_tau * (d[q] - f[q]);  // inv_tau * (feq_f - f)
        d[q] = f[q] - d[q];
        fout[q] = coll;
    }
    if constexpr (kForced) {
#define LBG_PF(q) fout[q] = f[q] + fluid_w * (fout[q] + forcing<q>(cu_of<q>(ux, uy, uz), ux, uy, uz, F.x, F.y, F.z))
        LBG_PF(0); LBG_PF(1); LBG_PF(2); LBG_PF(3); LBG_PF(4); LBG_PF(5); LBG_PF(6);
        LBG_PF(7); LBG_PF(8); LBG_PF(9); LBG_PF(10); LBG_PF(11); LBG_PF(12);
        LBG_PF(13); LBG_PF(14); LBG_PF(15); LBG_PF(16); LBG_PF(17); LBG_PF(18);
#undef LBG_PF
    } else {
#pragma unroll
        for (int q = 0; q < kQ; ++q) fout[q] = f[q] + fluid_w * fout[q];
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {  // static entry index keeps be/ue/m_out in registers
        if (e >= cnt) break;
        double fp[kQ];
        feq_all(rho, ue[e][0], ue[e][1], ue[e][2], fp);
        double mx = 0.0, my = 0.0, mz = 0.0;
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
            const double c_solid = d[opposite(q)] - (f[q] - fp[q]);
            fout[q] += be[e] * c_solid;
            // c_q = 0 terms subtract a signed zero from a sum that starts at +0 and
            // can never become -0 (x - x is +0), so they are skipped exactly
            if (cx(q) != 0) mx -= c_solid * (double)cx(q);
            if (cy(q) != 0) my -= c_solid * (double)cy(q);
            if (cz(q) != 0) mz -= c_solid * (double)cz(q);
        }
        m_out[e][0] = be[e] * mx;
        m_out[e][1] = be[e] * my;
        m_out[e][2] = be[e] * mz;
    }
#pragma unroll
    for (int q = 0; q < kQ; ++q) f[q] = fout[q];
    return ok;
}

// psm_cell for a cell with exactly one entry, scheduled pair by pair: everything direction
// q needs (f_q, feq_q, d_q̄, fp_q) lives in the (q, q̄) pair, so the output populations are
// produced and stored pair by pair instead of being held in registers. Same arithmetic as
// psm_cell_opt term for term (psm.cpp:174-216 with cnt == 1); the momentum sum keeps the q
// order because pairs are visited in q order. Returns ok; m_out = B * sum C c_qbar.
template <bool kForced>
__device__ __forceinline__ bool psm_cell_one(const double (&f)[kQ], double inv_tau, Force F,
                                             double b_tot, double be, double vx, double vy, double vz,
                                             double* __restrict__ dst, long long plane, long long base,
                                             double (&m_out)[3]) {
    double rho, ux, uy, uz;
    moments(f, rho, ux, uy, uz);
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const bool ok = rho > 0.0 && usq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    const double T = (0.5 * usq) * 3.0;
    const double Tp = (0.5 * ((vx * vx + vy * vy) + vz * vz)) * 3.0;
    const double fluid_w = 1.0 - b_tot;
    double mx = 0.0, my = 0.0, mz = 0.0;
    // fout_q = (f_q + w_f * (inv_tau * (feq_q - f_q) [+ F_q])) + B * ((f_qb - feq_qb) - (f_q - fp_q))
    auto out = [&](int q, double fq, double feq_q, double fqb, double feq_qb, double fp_q, double force) {
        const double coll = inv_tau * (feq_q - fq);
        const double base_out = fq + fluid_w * (kForced ? coll + force : coll);
        const double c_solid = (fqb - feq_qb) - (fq - fp_q);
        if (cx(q) != 0) mx -= c_solid * (double)cx(q);  // c_q = 0 terms are exact no-ops
        if (cy(q) != 0) my -= c_solid * (double)cy(q);
        if (cz(q) != 0) mz -= c_solid * (double)cz(q);
        dst[q * plane + base] = base_out + be * c_solid;
    };
    {
        const double feq0 = wq(0) * (rho - T);
        const double fp0 = wq(0) * (rho - Tp);
        out(0, f[0], feq0, f[0], feq0, fp0, kForced ? forcing<0>(0.0, ux, uy, uz, F.x, F.y, F.z) : 0.0);
    }
#define LBG_PAIR(qa, qb, cuf, cup)                                                                   \
    {                                                                                                \
        double fa, fb, pa, pb;                                                                       \
        feq_pair(wq(qa), (cuf), rho, T, fa, fb);                                                     \
        feq_pair(wq(qa), (cup), rho, Tp, pa, pb);                                                    \
        const double cu_a = (cuf);                                                                   \
        out(qa, f[qa], fa, f[qb], fb, pa, kForced ? forcing<qa>(cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0); \
        out(qb, f[qb], fb, f[qa], fa, pb, kForced ? forcing<qb>(-cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0); \
    }
    LBG_PAIR(1, 2, ux, vx)
    LBG_PAIR(3, 4, uy, vy)
    LBG_PAIR(5, 6, uz, vz)
    LBG_PAIR(7, 8, ux + uy, vx + vy)
    LBG_PAIR(9, 10, ux - uy, vx - vy)
    LBG_PAIR(11, 12, ux + uz, vx + vz)
    LBG_PAIR(13, 14, ux - uz, vx - vz)
    LBG_PAIR(15, 16, uy + uz, vy + vz)
    LBG_PAIR(17, 18, uy - uz, vy - vz)
#undef LBG_PAIR
    m_out[0] = be * mx;
    m_out[1] = be * my;
    m_out[2] = be * mz;
    return ok;
}

}  // namespace lbg
