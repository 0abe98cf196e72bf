// SPDX-License-Identifier: Apache-2.0
//
// Phase scheduler of the drop-in (a coupled step is 3j + 2 = 32 host phases,
// each closed by a barrier). The reference's ThreadPoolScheduler (partition.cpp:149-206) hands
// every phase to its workers through a mutex + condition variables: a futex wake of each
// worker and of the main thread per phase, tens of microseconds each. SpinPhaseScheduler keeps
// its contract exactly — block b runs on worker b % workers, run_phase returns when every
// worker finished the phase, the first exception of a phase is rethrown by run_phase — but
// publishes the phase through an atomic epoch that idle workers (and the waiting main thread)
// spin on for a bounded time before they block on the condition variable, so back-to-back
// phases start within a microsecond. Same work per block in the same order on the same thread:
// results are unchanged (LBDEM_GPU_SPIN_PHASES=0 keeps the reference's scheduler).
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <pthread.h>
#include <sched.h>

#include "lbdem/partition.hpp"

#if defined(__x86_64__) || defined(__i386__)
#include <immintrin.h>
#define LBDEM_CPU_RELAX() _mm_pause()
#else
#define LBDEM_CPU_RELAX() ((void)0)
#endif

namespace lbdem::gpu {

class SpinPhaseScheduler final : public partition::Scheduler {
public:
    /// spin_us: how long an idle thread polls before it blocks
    /// pin_stride > 0: worker w pinned to CPU (w * pin_stride) mod the CPU count (A/B)
    /// Spinning needs a CPU per spinning thread: a polling thread on an oversubscribed host
    /// holds the CPU a worker with work is waiting for (config 3 with 16 workers and the main
    /// thread all polling on 16 CPUs: ~100 ms per step instead of ~10). So the workers poll
    /// only when each can have a CPU of this process's affinity mask, and the main thread
    /// only when there is one more; otherwise they block right away, like the reference's.
    explicit SpinPhaseScheduler(int workers, int spin_us = 2000, int pin_stride = 0)
        : nw_(workers),
          spin_(std::chrono::microseconds(workers <= usable_cpus() ? spin_us : 0)),
          spin_main_(std::chrono::microseconds(workers + 1 <= usable_cpus() ? spin_us : 0)) {
        threads_.reserve(workers);
        for (int w = 0; w < workers; ++w) threads_.emplace_back([this, w] { worker_loop(w); });
        const int ncpu = static_cast<int>(std::thread::hardware_concurrency());
        if (pin_stride > 0 && ncpu > 0)
            for (int w = 0; w < workers; ++w) {
                cpu_set_t set;
                CPU_ZERO(&set);
                CPU_SET((w * pin_stride) % ncpu, &set);
                pthread_setaffinity_np(threads_[w].native_handle(), sizeof(set), &set);
            }
    }

    ~SpinPhaseScheduler() override {
        {
            std::lock_guard<std::mutex> lock(m_);
            stop_.store(true, std::memory_order_release);
        }
        cv_work_.notify_all();
        for (auto& t : threads_) t.join();
    }

    void run_phase(int n_blocks, const std::function<void(int)>& fn) override {
        fn_ = &fn;
        n_blocks_ = n_blocks;
        remaining_.store(nw_, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> lock(m_);  // a worker between its check and its wait sees it
            epoch_.fetch_add(1, std::memory_order_release);
        }
        cv_work_.notify_all();
        if (!spin_until([&] { return remaining_.load(std::memory_order_acquire) == 0; }, spin_main_)) {
            std::unique_lock<std::mutex> lock(m_);
            cv_main_.wait(lock, [&] { return remaining_.load(std::memory_order_acquire) == 0; });
        }
        fn_ = nullptr;
        if (error_) {
            std::exception_ptr e = error_;
            error_ = nullptr;
            std::rethrow_exception(e);
        }
    }

    int workers() const override { return nw_; }

    /// CPUs of this process's affinity mask (hardware_concurrency if unknown)
    static int usable_cpus() {
        cpu_set_t set;
        CPU_ZERO(&set);
        if (sched_getaffinity(0, sizeof(set), &set) == 0) return CPU_COUNT(&set);
        const int n = static_cast<int>(std::thread::hardware_concurrency());
        return n > 0 ? n : 1;
    }

    bool spinning() const { return spin_.count() > 0; }
    bool main_spinning() const { return spin_main_.count() > 0; }

private:
    template <class Pred>
    bool spin_until(Pred&& done, std::chrono::steady_clock::duration budget) const {
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0;; ++i) {
            if (done()) return true;
            LBDEM_CPU_RELAX();
            if ((i & 255) == 255 && std::chrono::steady_clock::now() - t0 > budget) return done();
        }
    }

    void worker_loop(int w) {
        long seen = 0;
        const int nw = nw_;  // (threads_ is still being filled while the first workers start)
        for (;;) {
            auto ready = [&] {
                return stop_.load(std::memory_order_acquire) || epoch_.load(std::memory_order_acquire) > seen;
            };
            if (!spin_until(ready, spin_)) {
                std::unique_lock<std::mutex> lock(m_);
                cv_work_.wait(lock, ready);
            }
            if (stop_.load(std::memory_order_acquire)) return;
            seen = epoch_.load(std::memory_order_acquire);
            const std::function<void(int)>* fn = fn_;
            const int n_blocks = n_blocks_;
            std::exception_ptr err;
            try {
                for (int b = w; b < n_blocks; b += nw) (*fn)(b);
            } catch (...) {
                err = std::current_exception();
            }
            if (err) {
                std::lock_guard<std::mutex> lock(m_);
                if (!error_) error_ = err;
            }
            if (remaining_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
                std::lock_guard<std::mutex> lock(m_);  // the main thread between its check and its wait
                cv_main_.notify_one();
            }
        }
    }

    const int nw_;
    std::vector<std::thread> threads_;
    std::mutex m_;
    std::condition_variable cv_main_, cv_work_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_blocks_ = 0;
    std::atomic<long> epoch_{0};
    std::atomic<int> remaining_{0};
    std::atomic<bool> stop_{false};
    std::exception_ptr error_;
    std::chrono::steady_clock::duration spin_;       // workers' poll budget
    std::chrono::steady_clock::duration spin_main_;  // the main thread's
};

}  // namespace lbdem::gpu
