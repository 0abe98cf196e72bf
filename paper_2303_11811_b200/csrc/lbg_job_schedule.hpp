// SPDX-License-Identifier: Apache-2.0
//
// The streamed host job's operation sequence (lbg_run_host, lbg_job.cu), host-only so a CPU test
// can replay it against the double-buffer semantics (tests/cpp/job_schedule_check.cpp):
//   Upload(z0, z1)   H2D of reference-layout planes [z0, z1) into the upload buffer A
//   Sweep(s, z0, z1) step s over planes [z0, z1): reads step s-1's buffer, writes step s's
//   Seam(s)          (z-slab decomposition) step s-1's planes 0 and nz-1 to the neighbours'
//                    z ghosts before step s's seam planes are swept (NCCL halo)
//   Download(z0, z1) D2H of the final step's planes [z0, z1) (at most `slab` planes)
// in the order the ops are enqueued on the compute stream. With planes [0, U) uploaded, step s
// is computable on [s, U - s); each step advances a frontier F[s] to U - s; once the last slab
// is in, every step in order completes [F[s], nz) and the seam planes [0, s).
#pragma once

#include <algorithm>
#include <vector>

namespace lbg::job {

enum class Op { Upload, Sweep, Seam, Download };

struct Item {
    Op op;
    int s;       // step (Sweep, Seam); 0 otherwise
    int z0, z1;  // plane range
};

// tail_split: the last slab's planes are uploaded in pieces of max(1, H / tail_split) — the
// planes whose final step waits for the last upload (the last piece plus the 2 x steps seam
// cone) are what goes down after the upload has ended, so a thinner last piece shortens that
// D2H-only tail (0 or 1: whole slabs throughout)
inline std::vector<Item> schedule(int nz, int steps, int slab, bool seam_halo, int tail_split = 0) {
    std::vector<Item> ops;
    if (nz <= 0 || steps < 0) return ops;
    const int H = std::max(1, std::min(slab, nz));
    auto download = [&](int z0, int z1) {
        for (int a = z0; a < z1; a += H) ops.push_back({Op::Download, 0, a, std::min(z1, a + H)});
    };
    std::vector<int> F(steps + 1);
    for (int s = 0; s <= steps; ++s) F[s] = s;
    F[0] = 0;
    int dl_next = steps;  // the next final plane to download in the main phase
    std::vector<int> ends;  // upload chunk ends
    const int tail0 = tail_split > 1 && nz > H ? nz - H : nz;
    for (int z = H; z < tail0; z += H) ends.push_back(z);
    if (tail0 < nz) {
        if (ends.empty() || ends.back() != tail0) ends.push_back(tail0);
        const int hs = std::max(1, H / tail_split);
        for (int z = tail0 + hs; z < nz; z += hs) ends.push_back(z);
    }
    ends.push_back(nz);
    for (size_t c = 0; c < ends.size(); ++c) {
        const int z0 = c == 0 ? 0 : ends[c - 1], z1 = ends[c];
        ops.push_back({Op::Upload, 0, z0, z1});
        F[0] = z1;
        if (z1 < nz) {
            for (int s = 1; s <= steps; ++s) {
                const int nf = z1 - s;
                if (nf > F[s]) {
                    ops.push_back({Op::Sweep, s, F[s], nf});
                    F[s] = nf;
                }
            }
            if (F[steps] > dl_next) {
                download(dl_next, F[steps]);
                dl_next = F[steps];
            }
        } else {
            for (int s = 1; s <= steps; ++s) {
                if (seam_halo) ops.push_back({Op::Seam, s, 0, 0});
                if (std::min(F[s], nz) < nz) ops.push_back({Op::Sweep, s, std::min(F[s], nz), nz});
                if (std::min(s, nz) > 0) ops.push_back({Op::Sweep, s, 0, std::min(s, nz)});
                F[s] = nz;
            }
            if (dl_next < nz) download(dl_next, nz);
            download(0, std::min(steps, nz));
        }
    }
    return ops;
}

}  // namespace lbg::job
