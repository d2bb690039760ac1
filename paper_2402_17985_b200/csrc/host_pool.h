// host_pool.h — a small persistent host thread pool (parallel_for) for the
// drop-in host path: staging pageable buffers through pinned bounce buffers
// (one thread's memcpy, ~10 GB/s, is well below PCIe gen5) and hashing recipe
// contents for the C++ shim's layer cache.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace fqg {

class HostPool {
   public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    int threads() const { return static_cast<int>(workers_.size()) + 1; }
    // fn(part) for part in [0, parts), on the workers and the calling thread.
    void parallel_for(int parts, const std::function<void(int)>& fn) {
        if (parts <= 1 || workers_.empty()) {
            for (int p = 0; p < parts; ++p) fn(p);
            return;
        }
        std::lock_guard<std::mutex> one(call_mu_);
        auto job = std::make_shared<Job>();
        job->fn = &fn;
        job->parts = parts;
        job->remaining.store(parts);
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = job;
            ++gen_;
        }
        cv_.notify_all();
        run(*job);
        std::unique_lock<std::mutex> lk(job->mu);
        job->done.wait(lk, [&] { return job->remaining.load() == 0; });
        job->fn = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

   private:
    struct Job {
        const std::function<void(int)>* fn = nullptr;
        int parts = 0;
        std::atomic<int> next{0}, remaining{0};
        std::mutex mu;
        std::condition_variable done;
    };
    HostPool() {
        const int n = std::clamp(static_cast<int>(std::thread::hardware_concurrency()) / 2, 1, 8);
        for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    static void run(Job& j) {
        for (;;) {
            const int p = j.next.fetch_add(1);
            if (p >= j.parts) return;  // (a late worker finds no part left)
            (*j.fn)(p);
            if (j.remaining.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> lk(j.mu);
                j.done.notify_all();
            }
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::shared_ptr<Job> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                job = job_;
            }
            run(*job);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_;
    std::shared_ptr<Job> job_;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

inline void parallel_copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t{1} << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const int parts = 4 * HostPool::get().threads();
    const size_t per = (bytes / parts + 63) & ~size_t{63};
    HostPool::get().parallel_for(parts, [&](int p) {
        const size_t b0 = std::min(bytes, per * static_cast<size_t>(p));
        const size_t b1 = p + 1 == parts ? bytes : std::min(bytes, b0 + per);
        if (b1 > b0)
            std::memcpy(static_cast<char*>(dst) + b0, static_cast<const char*>(src) + b0, b1 - b0);
    });
}

}  // namespace fqg
