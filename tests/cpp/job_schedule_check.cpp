// The streamed host job's schedule (paper_2303_11811_b200/csrc/lbg_job_schedule.hpp) replayed
// against the double-buffer semantics of lbg_run_host, for many (nz, steps, slab, seam) cases:
//   * a sweep of step s reads, for every plane it computes and its z neighbours, step s-1's
//     value from step s-1's buffer (A holds step 0 = the upload; neighbours across z = 0 /
//     nz - 1 wrap, or — with the NCCL seam — come from a Seam op issued for step s while
//     planes 0 and nz - 1 of step s-1's buffer held step s-1);
//   * every (step, plane) is computed exactly once, every plane uploaded once before use;
//   * every plane is downloaded exactly once, holding the final step, and no later op writes a
//     plane of the final buffer that was already queued for download (the pack reads it on
//     another stream); downloads are at most `slab` planes.
// Exit code != 0 names the first failed check.
#include <cstdio>
#include <vector>

#include "lbg_job_schedule.hpp"

using lbg::job::Item;
using lbg::job::Op;

static int check(int nz, int steps, int slab, bool seam, int tail = 0) {
    const std::vector<Item> ops = lbg::job::schedule(nz, steps, slab, seam, tail);
    const int H = slab < 1 ? 1 : (slab > nz ? nz : slab);
    std::vector<int> val[2] = {std::vector<int>(nz, -1), std::vector<int>(nz, -1)};  // step held, -1 none
    std::vector<int> uploaded(nz, 0), downloaded(nz, 0), queued(nz, 0);
    std::vector<std::vector<int>> computed(steps + 1, std::vector<int>(nz, 0));
    std::vector<int> seam_ok(steps + 1, 0);
    const int fin = steps & 1;
    for (const Item& it : ops) {
        switch (it.op) {
            case Op::Upload:
                for (int p = it.z0; p < it.z1; ++p) {
                    if (uploaded[p]++ || val[0][p] != -1) return 1;
                    val[0][p] = 0;
                }
                break;
            case Op::Seam: {
                const int src = (it.s - 1) & 1;
                if (!seam || val[src][0] != it.s - 1 || val[src][nz - 1] != it.s - 1) return 2;
                seam_ok[it.s] = 1;
                break;
            }
            case Op::Sweep: {
                const int s = it.s, src = (s - 1) & 1, dst = s & 1;
                if (s < 1 || s > steps || it.z0 < 0 || it.z1 > nz || it.z0 >= it.z1) return 3;
                for (int p = it.z0; p < it.z1; ++p) {
                    for (int d = -1; d <= 1; ++d) {
                        const int q = p + d;
                        if (q < 0 || q >= nz) {
                            if (seam) {
                                if (!seam_ok[s]) return 4;
                            } else if (val[src][(q + nz) % nz] != s - 1) {
                                return 5;
                            }
                        } else if (val[src][q] != s - 1) {
                            return 6;
                        }
                    }
                }
                for (int p = it.z0; p < it.z1; ++p) {
                    if (dst == fin && queued[p]) return 7;  // the pack may still be reading it
                    val[dst][p] = s;
                    if (computed[s][p]++) return 8;
                }
                break;
            }
            case Op::Download:
                if (it.z1 - it.z0 > H || it.z0 >= it.z1) return 9;
                for (int p = it.z0; p < it.z1; ++p) {
                    if (val[fin][p] != steps || downloaded[p]++) return 10;
                    queued[p] = 1;
                }
                break;
        }
    }
    for (int p = 0; p < nz; ++p) {
        if (!uploaded[p] || downloaded[p] != 1) return 11;
        for (int s = 1; s <= steps; ++s)
            if (computed[s][p] != 1) return 12;
    }
    return 0;
}

int main() {
    long cases = 0;
    for (int nz = 1; nz <= 40; ++nz)
        for (int steps = 0; steps <= 24; ++steps)
            for (int slab : {1, 2, 3, 4, 5, 7, 8, 16, 40, 64})
                for (int seam = 0; seam <= 1; ++seam)
                    for (int tail : {0, 4}) {
                        const int r = check(nz, steps, slab, seam != 0, tail);
                        ++cases;
                        if (r) {
                            std::printf("fail %d: nz=%d steps=%d slab=%d seam=%d tail=%d\n", r, nz, steps, slab, seam,
                                        tail);
                            return r;
                        }
                    }
    for (int steps : {0, 1, 20, 64})  // the benchmark's shape
        for (int seam = 0; seam <= 1; ++seam)
            if (int r = check(512, steps, 16, seam != 0, 4)) {
                std::printf("fail %d: nz=512 steps=%d\n", r, steps);
                return r;
            }
    std::printf("ok %ld\n", cases);
    return 0;
}
