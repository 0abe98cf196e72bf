// SPDX-License-Identifier: Apache-2.0
//
// K6 — periodic ghost fill  (fill_periodic_ghosts, boundary.cpp:98-137)
// K5 — domain-face BC fill   (apply_boundaries / fill_face, boundary.cpp:32-96, 140-146)
//
// Both write only ghost slots of the SOURCE buffer and read only interior cells, so one
// launch per operator covers all faces/regions:
//   * K6 enumerates the ghost shell (z planes, then y rows, then x columns) with one thread
//     per ghost cell. Each of the 26 regions is a wrap copy from an interior slab; they are
//     disjoint, so order does not matter. `full` copies all 19 q (bitwise-identical src
//     buffer); otherwise only the slots a pull sweep reads (g + c_q interior): 5 q per face
//     cell, 1 q per edge cell, none for corners — 5/19 of the traffic.
//   * K5 enumerates the (n+2)^2 ghost ring of every touching non-periodic face. A ghost
//     slot on the edge of two such faces is written by both faces in the reference with
//     the same value (both see a multi-wall link and bounce back), so the lower face index
//     owns it and the other skips it.
// Bytes per launch are tiny next to the sweep (<1% at 512^3).
#include "lbg_internal.cuh"

namespace lbg {

struct GhostArgs {
    double* __restrict__ src;
    Layout L;
    int periodic[3];
    int full;
    int wrap[3];  // axes the sweep wraps in-kernel (lbg_set_periodic_wrap)
    long long nA, nB, nC;  // shell region sizes
};

__device__ __forceinline__ bool interior(const Layout& L, int i, int j, int k) {
    return i >= 0 && i < L.nx && j >= 0 && j < L.ny && k >= 0 && k < L.nz;
}

// t -> ghost cell coordinates of the shell of the (nx+2)(ny+2)(nz+2) box
__device__ __forceinline__ void shell_cell(const GhostArgs& a, long long t, int& i, int& j, int& k) {
    const Layout& L = a.L;
    if (t < a.nA) {  // z planes k = -1 and nz, full (nx+2)(ny+2)
        const long long per = (long long)(L.nx + 2) * (L.ny + 2);
        k = t < per ? -1 : L.nz;
        const long long r = t % per;
        i = (int)(r % (L.nx + 2)) - 1;
        j = (int)(r / (L.nx + 2)) - 1;
        return;
    }
    t -= a.nA;
    if (t < a.nB) {  // y rows j = -1 and ny over k in [0,nz), all i
        const long long per = (long long)(L.nx + 2) * L.nz;
        j = t < per ? -1 : L.ny;
        const long long r = t % per;
        i = (int)(r % (L.nx + 2)) - 1;
        k = (int)(r / (L.nx + 2));
        return;
    }
    t -= a.nB;  // x columns i = -1 and nx over j in [0,ny), k in [0,nz)
    const long long per = (long long)L.ny * L.nz;
    i = t < per ? -1 : L.nx;
    const long long r = t % per;
    j = (int)(r % L.ny);
    k = (int)(r / L.ny);
}

__global__ void __launch_bounds__(256) periodic_fill_kernel(const GhostArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.nA + a.nB + a.nC) return;
    const Layout& L = a.L;
    int g[3];
    shell_cell(a, t, g[0], g[1], g[2]);
    const int n[3] = {L.nx, L.ny, L.nz};
    int s[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const int off = g[d] == -1 ? -1 : (g[d] == n[d] ? 1 : 0);
        if (off != 0 && !a.periodic[d]) return;  // region not periodic in every offset axis
        s[d] = off == 0 ? g[d] : (off == 1 ? 0 : n[d] - 1);
    }
    const long long gi = L.idx(g[0], g[1], g[2]);
    const long long si = L.idx(s[0], s[1], s[2]);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        if (!a.full) {
            // pulled by cell g + c_q; along in-kernel-wrapped axes that cell always exists
            const int t0 = g[0] + cx(q), t1 = g[1] + cy(q), t2 = g[2] + cz(q);
            const bool in0 = a.wrap[0] || (t0 >= 0 && t0 < L.nx);
            const bool in1 = a.wrap[1] || (t1 >= 0 && t1 < L.ny);
            const bool in2 = a.wrap[2] || (t2 >= 0 && t2 < L.nz);
            if (!(in0 && in1 && in2)) continue;
        }
        a.src[q * L.plane + gi] = a.src[q * L.plane + si];
    }
}

struct BcArgs {
    double* __restrict__ src;
    Layout L;
    int kind[6];
    int touches[6];
    double uw[6][3];
    double rho[6];
    int faces[6];  // processed faces in order
    int nfaces;
    long long fstart[7];
    DeviceErrors* err;
};

// boundary.cpp:75-80
__device__ __forceinline__ void cell_velocity(const BcArgs& a, long long si, double& ux, double& uy,
                                              double& uz) {
    double m0 = 0.0, m1 = 0.0, m2 = 0.0;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const double v = a.src[q * a.L.plane + si];
        m0 += (double)cx(q) * v;
        m1 += (double)cy(q) * v;
        m2 += (double)cz(q) * v;
    }
    ux = m0 / 1.0;
    uy = m1 / 1.0;
    uz = m2 / 1.0;
}

__global__ void __launch_bounds__(256) bc_fill_kernel(const BcArgs a) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.fstart[a.nfaces]) return;
    int fi = 0;
    while (t >= a.fstart[fi + 1]) ++fi;
    const int face = a.faces[fi];
    const Layout& L = a.L;
    const int n[3] = {L.nx, L.ny, L.nz};
    const int axis = face / 2, side = face % 2;
    // in-plane axes: the lower one varies fastest across threads (x for the y and z faces),
    // so a warp's ghost writes and interior reads walk along rows. The reference's visiting
    // order (jb outer, jc inner, boundary.cpp:94-95) is immaterial: each ghost slot of a face
    // is written once, and slots shared with another face go to the lower face (below).
    const int au = axis == 0 ? 1 : 0, av = axis == 2 ? 1 : 2;
    const long long r = t - a.fstart[fi];
    int g[3];
    g[axis] = side == 0 ? -1 : n[axis];
    g[au] = (int)(r % (n[au] + 2)) - 1;
    g[av] = (int)(r / (n[au] + 2)) - 1;

    // multi-wall flags per other axis, and edge ownership by the lower processed face
    bool multi_lo[3] = {false, false, false}, multi_hi[3] = {false, false, false};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (d == axis) continue;
        const bool wlo = a.touches[2 * d] && a.kind[2 * d] != LBG_BC_PERIODIC;
        const bool whi = a.touches[2 * d + 1] && a.kind[2 * d + 1] != LBG_BC_PERIODIC;
        multi_lo[d] = g[d] == -1 && wlo;
        multi_hi[d] = g[d] == n[d] && whi;
        // the same ghost slot belongs to face 2d / 2d+1 too; lower face index writes it
        if (multi_lo[d] && 2 * d < face) return;
        if (multi_hi[d] && 2 * d + 1 < face) return;
    }
    const bool multi = multi_lo[0] || multi_lo[1] || multi_lo[2] || multi_hi[0] || multi_hi[1] ||
                       multi_hi[2];
    const int kind = a.kind[face];
    const long long gi = LBG_IDX(L.idx(g[0], g[1], g[2]), L.plane, a.err);
#pragma unroll
    for (int q = 1; q < kQ; ++q) {
        const int s0 = g[0] + cx(q), s1 = g[1] + cy(q), s2 = g[2] + cz(q);
        if (!(s0 >= 0 && s0 < n[0] && s1 >= 0 && s1 < n[1] && s2 >= 0 && s2 < n[2])) continue;
        const long long si = LBG_IDX(L.idx(s0, s1, s2), L.plane, a.err);
        const double out = a.src[opposite(q) * L.plane + si];
        double v;
        if (multi || kind == LBG_BC_NO_SLIP) {
            v = out;
        } else if (kind == LBG_BC_VELOCITY) {
            const double cu = ((double)cx(q) * a.uw[face][0] + (double)cy(q) * a.uw[face][1]) +
                              (double)cz(q) * a.uw[face][2];
            v = out + (((2.0 * wq(q)) * 1.0) * cu) * 3.0;  // boundary.cpp:74
        } else {                                          // pressure, boundary.cpp:75-81
            double ux, uy, uz;
            cell_velocity(a, si, ux, uy, uz);
            const double cu = ((double)cx(q) * ux + (double)cy(q) * uy) + (double)cz(q) * uz;
            const double uu = (ux * ux + uy * uy) + uz * uz;
            const double feq_even = wq(q) * (a.rho[face] + 1.0 * ((((0.5 * cu) * cu) * 9.0) - (0.5 * uu) * 3.0));
            v = -out + 2.0 * feq_even;
        }
        a.src[q * L.plane + gi] = v;
    }
}

}  // namespace lbg

using namespace lbg;

extern "C" {

lbg_status lbg_fill_periodic(lbg_block b, const int periodic[3], int full) {
    if (lbg_status s_ = aa_refuse(b, "lbg_fill_periodic")) return s_;
    if (!b || !periodic) return set_error(LBG_INVALID, "null argument");
    if (!periodic[0] && !periodic[1] && !periodic[2]) return LBG_OK;
    LBG_CUDA(cudaSetDevice(b->device));
    GhostArgs a{};
    a.src = b->src();
    a.L = b->L;
    for (int d = 0; d < 3; ++d) a.periodic[d] = periodic[d] != 0;
    a.full = full != 0;
    for (int d = 0; d < 3; ++d) a.wrap[d] = b->wrap[d];
    const Layout& L = b->L;
    a.nA = 2LL * (L.nx + 2) * (L.ny + 2);
    a.nB = 2LL * (L.nx + 2) * L.nz;
    a.nC = 2LL * L.ny * L.nz;
    const long long n = a.nA + a.nB + a.nC;
    Span span(b, LBG_CAT_PSM_COMM);
    periodic_fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

lbg_status lbg_apply_boundaries(lbg_block b, const lbg_face_bc faces[6], const int touches[6]) {
    if (lbg_status s_ = aa_refuse(b, "lbg_apply_boundaries")) return s_;
    if (!b || !faces || !touches) return set_error(LBG_INVALID, "null argument");
    // BcSpec::validate (boundary.cpp:8-16)
    for (int axis = 0; axis < 3; ++axis) {
        const bool lo = faces[2 * axis].kind == LBG_BC_PERIODIC;
        const bool hi = faces[2 * axis + 1].kind == LBG_BC_PERIODIC;
        if (lo != hi)
            return set_error(LBG_CONFIG_ERROR,
                             "periodic boundary must be assigned to both faces of axis " +
                                 std::to_string(axis));
    }
    BcArgs a{};
    a.src = b->src();
    a.L = b->L;
    a.err = b->err_d;
    const Layout& L = b->L;
    const int n[3] = {L.nx, L.ny, L.nz};
    a.fstart[0] = 0;
    for (int f = 0; f < 6; ++f) {
        a.kind[f] = faces[f].kind;
        a.touches[f] = touches[f] != 0;
        for (int c = 0; c < 3; ++c) a.uw[f][c] = faces[f].u_wall[c];
        a.rho[f] = faces[f].rho;
        if (!touches[f] || faces[f].kind == LBG_BC_PERIODIC) continue;
        const int axis = f / 2;
        const long long ring = (long long)(n[(axis + 1) % 3] + 2) * (n[(axis + 2) % 3] + 2);
        a.faces[a.nfaces] = f;
        a.fstart[a.nfaces + 1] = a.fstart[a.nfaces] + ring;
        ++a.nfaces;
    }
    if (a.nfaces == 0) return LBG_OK;
    LBG_CUDA(cudaSetDevice(b->device));
    const long long total = a.fstart[a.nfaces];
    Span span(b, LBG_CAT_OTHER);
    bc_fill_kernel<<<(unsigned)((total + 255) / 256), 256, 0, b->stream>>>(a);
    LBG_LAUNCH_CHECK();
    return LBG_OK;
}

}  // extern "C"
