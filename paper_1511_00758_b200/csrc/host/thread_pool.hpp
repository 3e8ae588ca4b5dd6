// thread_pool.hpp — fixed host worker pool for the per-frame Delaunay step.
// The reference's only concurrency is fork/join row bands
// (proj/include/planestereo/parallel.hpp:13-37); here the host parallelism is
// across frames of a batch, and results do not depend on the schedule.
#pragma once

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace ps {

class ThreadPool {
public:
    explicit ThreadPool(int threads) {
        if (threads < 1) threads = 1;
        for (int i = 0; i < threads - 1; ++i) workers_.emplace_back([this, i] { loop(i + 1); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++generation_;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    int size() const { return int(workers_.size()) + 1; }

    // Runs fn(item, worker) for item in [0, n); the caller participates as worker 0.
    void parallel_for(int n, const std::function<void(int, int)>& fn) {
        if (n <= 0) return;
        if (workers_.empty() || n == 1) {
            for (int i = 0; i < n; ++i) fn(i, 0);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            fn_ = &fn;
            n_ = n;
            next_.store(0);
            active_ = int(workers_.size());
            ++generation_;
        }
        cv_.notify_all();
        run_items(0);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [this] { return active_ == 0; });
        fn_ = nullptr;
    }

private:
    void run_items(int worker) {
        for (;;) {
            const int i = next_.fetch_add(1);
            if (i >= n_) break;
            (*fn_)(i, worker);
        }
    }
    void loop(int worker) {
        long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return generation_ != seen; });
                seen = generation_;
                if (stop_) return;
            }
            run_items(worker);
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--active_ == 0) done_cv_.notify_one();
            }
        }
    }

    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)>* fn_ = nullptr;
    int n_ = 0;
    std::atomic<int> next_{0};
    int active_ = 0;
    long long generation_ = 0;
    bool stop_ = false;
};

}  // namespace ps
