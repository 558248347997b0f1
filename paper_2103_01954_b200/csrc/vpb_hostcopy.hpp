// vpb_hostcopy.hpp — host-side staging for pageable caller memory (the drop-in path: the
// reference's Scene owns its slab in an ordinary std::vector). A CUDA copy from pageable memory
// runs through the driver's own bounce buffer at a fraction of PCIe speed, so large pageable
// transfers are staged here instead: a small pool of host threads copies the caller's bytes into
// page-locked chunks, while the copy engine moves the previous chunk to the device.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

namespace vpb {

// Fixed pool of workers splitting one memcpy at a time.
class CopyPool {
  public:
    // Throws (std::system_error) when a thread cannot be created; the threads started so far
    // are stopped and joined first.
    explicit CopyPool(int n_threads) {
        try {
            for (int i = 0; i < n_threads; ++i) workers_.emplace_back([this, i] { run(i); });
        } catch (...) {
            shutdown();
            throw;
        }
    }
    ~CopyPool() { shutdown(); }
    CopyPool(const CopyPool &) = delete;
    CopyPool &operator=(const CopyPool &) = delete;

    // memcpy(dst, src, bytes) split over the workers plus the calling thread.
    void copy(void *dst, const void *src, size_t bytes) {
        const int parts = int(workers_.size()) + 1;
        if (bytes < (size_t(1) << 20) || parts == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            dst_ = static_cast<unsigned char *>(dst);
            src_ = static_cast<const unsigned char *>(src);
            bytes_ = bytes;
            pending_ = int(workers_.size());
            ++gen_;
        }
        cv_.notify_all();
        slice(int(workers_.size()), parts);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void shutdown() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (std::thread &t : workers_) t.join();
        workers_.clear();
    }
    void slice(int i, int parts) const {
        const size_t per = (bytes_ / size_t(parts) + 4095) & ~size_t(4095);
        const size_t lo = std::min(bytes_, per * size_t(i)), hi = std::min(bytes_, lo + per);
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void run(int i) {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            slice(i, int(workers_.size()) + 1);
            {
                std::lock_guard<std::mutex> g(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }

    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    unsigned long long gen_ = 0;
    bool stop_ = false;
    int pending_ = 0;
    unsigned char *dst_ = nullptr;
    const unsigned char *src_ = nullptr;
    size_t bytes_ = 0;
};

}  // namespace vpb
