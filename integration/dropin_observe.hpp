// SPDX-License-Identifier: Apache-2.0
//
// Drop-in observers: the reference's per-cell walks over the host PdfField
// (lbm::cell_macroscopic / total_mass / total_momentum, lbm.cpp:61-93; io::sample_scalars /
// write_grid_dump, output.cpp:22-107) read a per-block cache of device moments instead —
// {rho, mx, my, mz, btot} per cell from lbg_moments, 40 B per cell over PCIe instead of the
// 152 B of populations plus the fraction field, and no host mirror needed.
//
// Every value the observers consume is the reference's own arithmetic: rho and the bare
// momentum are the device's bitwise per-cell sums; the compensated totals and the
// observable velocity u = m / rho0 + (dt / (2 rho0)) f_ext (lbm.hpp:62) are evaluated here,
// in the reference's loop order, so the results are bit-identical to the CPU solver's.
#pragma once

#include <vector>

#include "lbdem/lbm.hpp"
#include "lbdem/sim.hpp"
#include "lbdem/vec3.hpp"
#include "lbdem_gpu.hpp"

namespace lbdem::gpu {

/// The block's moments, refreshed from the device when a step has run since the last read.
inline const std::vector<double>& cell_moments(const BlockState& b) {
    if (b.moments_stale || b.moments.empty()) {
        b.dev->moments(b.moments);
        b.moments_stale = false;
    }
    return b.moments;
}

inline std::size_t cell_index(const BlockState& b, int i, int j, int k) {
    const Vec3i d = b.dims();
    return (static_cast<std::size_t>(k) * d.y + j) * d.x + i;
}

/// lbm::cell_macroscopic (lbm.cpp:61-67 -> lbm.hpp:55-63)
inline void cell_macroscopic(const BlockState& b, const Vec3& f_ext, int i, int j, int k,
                             double& rho, Vec3& u) {
    const double* m = cell_moments(b).data() + 5 * cell_index(b, i, j, k);
    rho = m[0];
    const Vec3 mom{m[1], m[2], m[3]};
    u = mom / lbm::kRho0 + (lbm::kDt / (2.0 * lbm::kRho0)) * f_ext;
}

/// FractionField::btot of an interior cell (0 for an uncoupled block), as write_grid_dump prints
inline double cell_fraction(const BlockState& b, int i, int j, int k) {
    return cell_moments(b)[5 * cell_index(b, i, j, k) + 4];
}

/// lbm::total_mass (lbm.cpp:69-80): compensated sum of rho in (k, j, i) order
inline double total_mass(const BlockState& b) {
    const std::vector<double>& m = cell_moments(b);
    CompensatedSum mass;
    for (std::size_t c = 0; c < m.size(); c += 5) mass.add(m[c]);
    return mass.value();
}

/// lbm::total_momentum (lbm.cpp:82-93): compensated sum of the bare momentum in (k, j, i) order
inline Vec3 total_momentum(const BlockState& b) {
    const std::vector<double>& m = cell_moments(b);
    CompensatedVec3 mom;
    for (std::size_t c = 0; c < m.size(); c += 5) mom.add(Vec3{m[c + 1], m[c + 2], m[c + 3]});
    return mom.value();
}

}  // namespace lbdem::gpu
