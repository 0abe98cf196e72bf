// SpinPhaseScheduler (integration/dropin_sched.hpp) against the ThreadPoolScheduler contract
// (partition.hpp:170-192): every block once per phase, block b always on worker b % workers,
// the phase's exception rethrown by run_phase, idle threads falling back to blocking, no
// spinning when the threads outnumber the CPUs.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <mutex>
#include <set>
#include <stdexcept>
#include <thread>
#include <vector>

#include "dropin_sched.hpp"

int main() {
    // fresh schedulers: the first phase may start while the later workers are still starting
    for (int rep = 0; rep < 200; ++rep) {
        lbdem::gpu::SpinPhaseScheduler s(8, 100);
        for (int p = 0; p < 3; ++p) {
            std::vector<std::atomic<int>> seen(8);
            s.run_phase(8, [&](int b) { seen[b].fetch_add(1); });
            for (int b = 0; b < 8; ++b)
                if (seen[b].load() != 1) return 7;
        }
    }
    const int workers = 4, blocks = 11, phases = 2000;
    lbdem::gpu::SpinPhaseScheduler s(workers, 200);
    if (s.workers() != workers) return 1;
    std::vector<std::thread::id> owner(blocks);
    std::vector<int> count(blocks, 0);
    std::mutex m;
    for (int p = 0; p < phases; ++p) {
        std::vector<std::atomic<int>> seen(blocks);
        s.run_phase(blocks, [&](int b) {
            seen[b].fetch_add(1);
            std::lock_guard<std::mutex> lock(m);
            if (p == 0) owner[b] = std::this_thread::get_id();
            else if (owner[b] != std::this_thread::get_id()) throw std::runtime_error("block moved to another worker");
            ++count[b];
        });
        for (int b = 0; b < blocks; ++b)
            if (seen[b].load() != 1) return 2;
        if (p % 500 == 0) std::this_thread::sleep_for(std::chrono::milliseconds(2));  // blocking path
    }
    for (int b = 0; b < blocks; ++b)
        if (count[b] != phases) return 3;
    for (int b = 0; b < blocks; ++b)
        for (int c = 0; c < blocks; ++c)
            if ((b % workers == c % workers) != (owner[b] == owner[c])) return 4;
    bool thrown = false;
    try {
        s.run_phase(blocks, [&](int b) {
            if (b == 7) throw std::runtime_error("phase error");
        });
    } catch (const std::runtime_error& e) {
        thrown = std::string(e.what()) == "phase error";
    }
    if (!thrown) return 5;
    int after = 0;  // the scheduler stays usable after an exception
    s.run_phase(blocks, [&](int) {
        std::lock_guard<std::mutex> lock(m);
        ++after;
    });
    if (after != blocks) return 6;
    // more threads than CPUs: no spinning (a polling thread would hold a working one's CPU),
    // and the contract still holds on the blocking path
    {
        const int ncpu = lbdem::gpu::SpinPhaseScheduler::usable_cpus();
        lbdem::gpu::SpinPhaseScheduler full(ncpu, 2000);  // a CPU per worker: workers poll, main blocks
        if (!full.spinning() || full.main_spinning()) return 11;
        lbdem::gpu::SpinPhaseScheduler over(ncpu + 1, 2000);
        if (over.spinning() || over.main_spinning()) return 8;
        std::vector<std::atomic<int>> seen(2 * ncpu);
        for (int p = 0; p < 50; ++p) over.run_phase(2 * ncpu, [&](int b) { seen[b].fetch_add(1); });
        for (int p = 0; p < 50; ++p) full.run_phase(2 * ncpu, [&](int b) { seen[b].fetch_add(1); });
        for (auto& v : seen)
            if (v.load() != 100) return 9;
        if (ncpu >= 2 && !lbdem::gpu::SpinPhaseScheduler(ncpu - 1, 2000).main_spinning()) return 10;
    }
    std::printf("ok\n");
    return 0;
}
