// thread_pool.hpp — fixed host worker pool for the per-frame Delaunay step.
// The reference's only concurrency is fork/join row bands
// (proj/include/planestereo/parallel.hpp:13-37); here the host parallelism is
// across frames of a batch, and results do not depend on the schedule.
//
// Two modes: submit() queues independent tasks (the engine's dataflow loop
// keeps the workers busy while it launches device work), parallel_for() runs
// n items and returns when all are done.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace ps {

class ThreadPool {
public:
    explicit ThreadPool(int threads) {
        if (threads < 1) threads = 1;
        for (int i = 0; i < threads; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    int size() const { return int(workers_.size()); }

    // Queues fn(worker); returns immediately.
    void submit(std::function<void(int)> fn) {
        {
            std::lock_guard<std::mutex> lk(m_);
            q_.push_back(std::move(fn));
            ++outstanding_;
        }
        cv_.notify_one();
    }

    // Blocks until every submitted task has finished.
    void wait_idle() {
        std::unique_lock<std::mutex> lk(m_);
        idle_cv_.wait(lk, [this] { return outstanding_ == 0; });
    }

    // Runs fn(item, worker) for item in [0, n) and waits for completion.
    void parallel_for(int n, const std::function<void(int, int)>& fn) {
        if (n <= 0) return;
        for (int i = 0; i < n; ++i) submit([&fn, i](int w) { fn(i, w); });
        wait_idle();
    }

    // Runs fn(item, worker) for item in [0, n) from inside a task running on
    // `self`: the caller works through the items itself while up to n - 1
    // helper tasks (queued behind earlier tasks) take items in parallel when
    // a worker is free.  Returns when every item has finished; a helper that
    // starts after that finds no item and returns without touching fn.
    void help_run(int self, int n, const std::function<void(int, int)>& fn) {
        if (n <= 0) return;
        struct State {
            std::atomic<int> next{0};
            int done = 0;
            std::mutex m;
            std::condition_variable cv;
        };
        auto st = std::make_shared<State>();
        // fn is alive while an item is unclaimed (the caller waits for all)
        auto work = [st, n](int w, const std::function<void(int, int)>* f) {
            for (int i; (i = st->next.fetch_add(1)) < n;) {
                (*f)(i, w);
                std::lock_guard<std::mutex> lk(st->m);
                if (++st->done == n) st->cv.notify_all();
            }
        };
        const int helpers = std::min(n - 1, size() - 1);
        const std::function<void(int, int)>* fp = &fn;
        for (int h = 0; h < helpers; ++h)
            submit([st, n, work, fp](int w) {
                if (st->next.load() < n) work(w, fp);
            });
        work(self, fp);
        std::unique_lock<std::mutex> lk(st->m);
        st->cv.wait(lk, [&] { return st->done == n; });
    }

private:
    void loop(int worker) {
        for (;;) {
            std::function<void(int)> task;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                task = std::move(q_.front());
                q_.pop_front();
            }
            task(worker);
            {
                std::lock_guard<std::mutex> lk(m_);
                if (--outstanding_ == 0) idle_cv_.notify_all();
            }
        }
    }

    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, idle_cv_;
    std::deque<std::function<void(int)>> q_;
    long long outstanding_ = 0;
    bool stop_ = false;
};

}  // namespace ps
