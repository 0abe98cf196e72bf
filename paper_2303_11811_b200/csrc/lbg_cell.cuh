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
// psm_cell_one / psm_cell_two: the covered-cell operator (psm.cpp:174-216) for one or two
// entries, scheduled pair by pair (q, opposite q) so no direction's output is held in a
// register past its pair; the per-direction and momentum operation orders are the
// reference's (the oracle restates the literal form, oracle/lbm_oracle.c).
#pragma once

#include "lbg_internal.cuh"

namespace lbg {

// PDF stores of the fused operators. A/B builds (-DLBG_STORE_CS) use the streaming store
// (st.global.cs: evict-first), so the stored populations do not displace the coupling fields
// and snapshots from L1/L2.
__device__ __forceinline__ void pdf_store(double* p, double v) {
#ifdef LBG_STORE_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}


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

// psm_cell for a cell with exactly one entry, scheduled pair by pair: everything direction
// q needs (f_q, feq_q, d_q̄, fp_q) lives in the (q, q̄) pair, so the output populations are
// produced and stored pair by pair instead of being held in registers. Same arithmetic as
// psm_cell (psm.cpp:174-216 with cnt == 1) term for term, the fluid equilibrium entering as
// d = f - feq (feq - f == -d exactly); the momentum sum keeps the q
// order because pairs are visited in q order. Returns ok; m_out = B * sum C c_qbar.
template <bool kForced, class Get>
__device__ __forceinline__ void psm_one_pairs_g(Get f, double rho, double ux, double uy, double uz, double usq,
                                                double inv_tau, Force F, double b_tot, double be, double vx,
                                                double vy, double vz, double* __restrict__ dst, long long plane,
                                                long long base, double (&m_out)[3]);

template <bool kForced>
__device__ __forceinline__ void psm_cell_one_pairs(const double (&f)[kQ], double rho, double ux, double uy,
                                                   double uz, double usq, double inv_tau, Force F, double b_tot,
                                                   double be, double vx, double vy, double vz,
                                                   double* __restrict__ dst, long long plane, long long base,
                                                   double (&m_out)[3]) {
    psm_one_pairs_g<kForced>([&](int q) { return f[q]; }, rho, ux, uy, uz, usq, inv_tau, F, b_tot, be, vx, vy, vz,
                             dst, plane, base, m_out);
}

template <bool kForced>
__device__ __forceinline__ bool psm_cell_one(const double (&f)[kQ], double inv_tau, Force F,
                                             double b_tot, double be, double vx, double vy, double vz,
                                             double* __restrict__ dst, long long plane, long long base,
                                             double (&m_out)[3]) {
    double rho, ux, uy, uz;
    moments(f, rho, ux, uy, uz);
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const bool ok = rho > 0.0 && usq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    psm_cell_one_pairs<kForced>(f, rho, ux, uy, uz, usq, inv_tau, F, b_tot, be, vx, vy, vz, dst, plane, base,
                                m_out);
    return ok;
}

// psm_cell_one after the moments: the pair-by-pair outputs and the entry's momentum. f(q)
// yields population q: a register of the pulled array, or (low-register kernels) a re-read of
// the pulled value from L1.
template <bool kForced, class Get>
__device__ __forceinline__ void psm_one_pairs_g(Get f, double rho, double ux, double uy, double uz, double usq,
                                                double inv_tau, Force F, double b_tot, double be, double vx,
                                                double vy, double vz, double* __restrict__ dst, long long plane,
                                                long long base, double (&m_out)[3]) {
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
        pdf_store(dst + q * plane + base, base_out + be * c_solid);
    };
    {
        const double f0 = f(0);
        const double feq0 = wq(0) * (rho - T);
        const double fp0 = wq(0) * (rho - Tp);
        out(0, f0, feq0, f0, feq0, fp0, kForced ? forcing<0>(0.0, ux, uy, uz, F.x, F.y, F.z) : 0.0);
    }
#define LBG_PAIR(qa, qb, cuf, cup)                                                                   \
    {                                                                                                \
        const double xa = f(qa), xb = f(qb);                                                         \
        double fa, fb, pa, pb;                                                                       \
        feq_pair(wq(qa), (cuf), rho, T, fa, fb);                                                     \
        feq_pair(wq(qa), (cup), rho, Tp, pa, pb);                                                    \
        const double cu_a = (cuf);                                                                   \
        out(qa, xa, fa, xb, fb, pa, kForced ? forcing<qa>(cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0);   \
        out(qb, xb, fb, xa, fa, pb, kForced ? forcing<qb>(-cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0);  \
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
}

// collide_cell (unforced) after the moments, pair by pair: the same operations as srt_cell
// (out = f + inv_tau * (feq - f), feq from feq_pair), f(q) as in psm_one_pairs_g
template <class Get>
__device__ __forceinline__ void srt_pairs_g(Get f, double rho, double ux, double uy, double uz, double usq,
                                            double inv_tau, double* __restrict__ dst, long long plane,
                                            long long base) {
    const double T = (0.5 * usq) * 3.0;
    {
        const double f0 = f(0);
        pdf_store(dst + base, f0 + inv_tau * (wq(0) * (rho - T) - f0));
    }
#define LBG_SPAIR(qa, qb, cuf)                                  \
    {                                                           \
        const double xa = f(qa), xb = f(qb);                    \
        double fa, fb;                                          \
        feq_pair(wq(qa), (cuf), rho, T, fa, fb);                \
        pdf_store(dst + qa * plane + base, xa + inv_tau * (fa - xa)); \
        pdf_store(dst + qb * plane + base, xb + inv_tau * (fb - xb)); \
    }
    LBG_SPAIR(1, 2, ux)
    LBG_SPAIR(3, 4, uy)
    LBG_SPAIR(5, 6, uz)
    LBG_SPAIR(7, 8, ux + uy)
    LBG_SPAIR(9, 10, ux - uy)
    LBG_SPAIR(11, 12, ux + uz)
    LBG_SPAIR(13, 14, ux - uz)
    LBG_SPAIR(15, 16, uy + uz)
    LBG_SPAIR(17, 18, uy - uz)
#undef LBG_SPAIR
}

// psm_cell for a cell with one or two entries, scheduled pair by pair like psm_cell_one
// (psm.cpp:174-216). Entry 1 enters only where `two` is set, so a one-entry (or, unforced,
// fluid: B = b = 0, v = 0) lane gets exactly psm_cell_one's result; per direction
// fout_q = ((f_q + w_f * (inv_tau * (feq_q - f_q) [+ F_q])) + b_0 * C_0q) + b_1 * C_1q, the
// order of psm_cell's entry loop (psm.cpp:198-214), and the two momentum sums run in q order.
template <bool kForced>
__device__ __forceinline__ bool psm_cell_two(const double (&f)[kQ], double inv_tau, Force F, double b_tot,
                                             double be0, const double (&v0)[3], double be1,
                                             const double (&v1)[3], bool two, double* __restrict__ dst,
                                             long long plane, long long base, double (&m_out)[2][3]) {
    double rho, ux, uy, uz;
    moments(f, rho, ux, uy, uz);
    const double usq = (ux * ux + uy * uy) + uz * uz;
    const bool ok = rho > 0.0 && usq <= kMaxVelocity * kMaxVelocity && isfinite(rho);
    const double T = (0.5 * usq) * 3.0;
    const double T0 = (0.5 * ((v0[0] * v0[0] + v0[1] * v0[1]) + v0[2] * v0[2])) * 3.0;
    const double T1 = (0.5 * ((v1[0] * v1[0] + v1[1] * v1[1]) + v1[2] * v1[2])) * 3.0;
    const double fluid_w = 1.0 - b_tot;
    double m0x = 0.0, m0y = 0.0, m0z = 0.0, m1x = 0.0, m1y = 0.0, m1z = 0.0;
    auto out = [&](int q, double fq, double feq_q, double fqb, double feq_qb, double p0_q, double p1_q,
                   double force) {
        const double coll = inv_tau * (feq_q - fq);
        const double base_out = fq + fluid_w * (kForced ? coll + force : coll);
        const double c0 = (fqb - feq_qb) - (fq - p0_q);
        const double c1 = (fqb - feq_qb) - (fq - p1_q);
        if (cx(q) != 0) m0x -= c0 * (double)cx(q);  // c_q = 0 terms are exact no-ops
        if (cy(q) != 0) m0y -= c0 * (double)cy(q);
        if (cz(q) != 0) m0z -= c0 * (double)cz(q);
        if (cx(q) != 0) m1x -= c1 * (double)cx(q);
        if (cy(q) != 0) m1y -= c1 * (double)cy(q);
        if (cz(q) != 0) m1z -= c1 * (double)cz(q);
        const double r0 = base_out + be0 * c0;
        pdf_store(dst + q * plane + base, two ? r0 + be1 * c1 : r0);
    };
    {
        const double feq0 = wq(0) * (rho - T);
        out(0, f[0], feq0, f[0], feq0, wq(0) * (rho - T0), wq(0) * (rho - T1),
            kForced ? forcing<0>(0.0, ux, uy, uz, F.x, F.y, F.z) : 0.0);
    }
#define LBG_PAIR2(qa, qb, cuf, cu0, cu1)                                                                  \
    {                                                                                                  \
        double fa, fb, pa0, pb0, pa1, pb1;                                                             \
        feq_pair(wq(qa), (cuf), rho, T, fa, fb);                                                       \
        feq_pair(wq(qa), (cu0), rho, T0, pa0, pb0);                                                    \
        feq_pair(wq(qa), (cu1), rho, T1, pa1, pb1);                                                    \
        const double cu_a = (cuf);                                                                     \
        out(qa, f[qa], fa, f[qb], fb, pa0, pa1, kForced ? forcing<qa>(cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0); \
        out(qb, f[qb], fb, f[qa], fa, pb0, pb1, kForced ? forcing<qb>(-cu_a, ux, uy, uz, F.x, F.y, F.z) : 0.0); \
    }
    LBG_PAIR2(1, 2, ux, v0[0], v1[0])
    LBG_PAIR2(3, 4, uy, v0[1], v1[1])
    LBG_PAIR2(5, 6, uz, v0[2], v1[2])
    LBG_PAIR2(7, 8, ux + uy, v0[0] + v0[1], v1[0] + v1[1])
    LBG_PAIR2(9, 10, ux - uy, v0[0] - v0[1], v1[0] - v1[1])
    LBG_PAIR2(11, 12, ux + uz, v0[0] + v0[2], v1[0] + v1[2])
    LBG_PAIR2(13, 14, ux - uz, v0[0] - v0[2], v1[0] - v1[2])
    LBG_PAIR2(15, 16, uy + uz, v0[1] + v0[2], v1[1] + v1[2])
    LBG_PAIR2(17, 18, uy - uz, v0[1] - v0[2], v1[1] - v1[2])
#undef LBG_PAIR2
    m_out[0][0] = be0 * m0x;
    m_out[0][1] = be0 * m0y;
    m_out[0][2] = be0 * m0z;
    m_out[1][0] = be1 * m1x;
    m_out[1][1] = be1 * m1y;
    m_out[1][2] = be1 * m1z;
    return ok;
}

}  // namespace lbg
