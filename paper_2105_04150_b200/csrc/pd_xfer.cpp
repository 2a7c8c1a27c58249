// pd_xfer.cpp -- host <-> device copies of the large arrays (rows, state).
//
// The caller's arrays are ordinary pageable std::vector storage.  Copying
// them with cudaMemcpyAsync from pageable memory runs at ~6 GB/s (the driver
// stages through a small internal buffer).  Here each copy is cut into 32 MB
// chunks that go through two pinned bounce buffers: several host threads fill
// (or drain) one buffer while the DMA engine moves the other, so a 5 GB row
// array crosses in ~0.25 s instead of ~0.8 s.  Copies below 8 MB go direct.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

#include "pd_internal.h"

namespace pdb {

namespace {

constexpr size_t kChunk = size_t(32) << 20;
constexpr size_t kDirect = size_t(8) << 20;
constexpr int kBuf = 3;  // bounce buffers: host fill, DMA and one spare in flight

struct Bounce {
    void* buf[kBuf] = {};
    cudaEvent_t done[kBuf] = {};
    int device = -1;
    ~Bounce() {
        for (int k = 0; k < kBuf; ++k) {
            if (buf[k])
                cudaFreeHost(buf[k]);
            if (done[k])
                cudaEventDestroy(done[k]);
        }
    }
    cudaError_t ensure() {
        int dev = 0;
        cudaGetDevice(&dev);
        if (buf[0] && device == dev)
            return cudaSuccess;
        for (int k = 0; k < kBuf; ++k) {
            if (!buf[k]) {
                cudaError_t e = cudaHostAlloc(&buf[k], kChunk, cudaHostAllocPortable);
                if (e != cudaSuccess)
                    return e;
            }
            if (done[k])
                cudaEventDestroy(done[k]);
            cudaError_t e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
            if (e != cudaSuccess)
                return e;
        }
        device = dev;
        return cudaSuccess;
    }
};

thread_local Bounce t_bounce;

// memcpy split over a persistent pool of host threads (one memcpy stream tops
// out near 10 GB/s).  A pool, not threads per call: a 5 GB row array is 160
// chunks, and spawning the workers for each chunk cost ~10 % of the copy.
// PD_XFER_THREADS overrides the worker count (default min(16, cores)).
class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* p = new CopyPool;  // never destroyed: workers outlive static teardown
        return *p;
    }
    void copy(void* dst, const void* src, size_t bytes) {
        const size_t parts = std::min<size_t>(size_t(workers_) + 1, bytes / (size_t(2) << 20) + 1);
        if (parts <= 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);  // one job at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            step_ = (bytes + parts - 1) / parts;
            next_ = 1;  // part 0 is the caller's
            parts_ = parts;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        run_part(0);
        for (;;) {  // help with the remaining parts, then wait for the workers
            const size_t k = claim();
            if (k >= parts)
                break;
            run_part(k);
            finish();
        }
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        int n = int(std::min(16u, hw)) - 1;
        if (const char* e = std::getenv("PD_XFER_THREADS"))
            n = std::max(0, std::atoi(e) - 1);
        workers_ = n;
        for (int t = 0; t < n; ++t)
            std::thread([this] { loop(); }).detach();
    }
    size_t claim() {
        std::lock_guard<std::mutex> lk(mu_);
        return next_ < parts_ ? next_++ : parts_;
    }
    void finish() {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0)
            done_cv_.notify_all();
    }
    void run_part(size_t k) {
        const size_t b = k * step_, e = std::min(bytes_, b + step_);
        if (b < e)
            std::memcpy(dst_ + b, src_ + b, e - b);
    }
    void loop() {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen && next_ < parts_; });
                seen = gen_;
            }
            for (;;) {
                const size_t k = claim();
                if (k >= parts_)
                    break;
                run_part(k);
                finish();
            }
        }
    }
    int workers_ = 0;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0, step_ = 0, next_ = 0, parts_ = 0, pending_ = 0;
    unsigned long long gen_ = 0;
};

void par_memcpy(void* dst, const void* src, size_t bytes) { CopyPool::get().copy(dst, src, bytes); }

} // namespace

cudaError_t h2d_large(void* dev, const void* host, size_t bytes, cudaStream_t s) {
    if (bytes < kDirect)
        return cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s);
    Bounce& B = t_bounce;
    cudaError_t e = B.ensure();
    if (e != cudaSuccess)
        return e;
    bool used[kBuf] = {};
    for (size_t off = 0, k = 0; off < bytes; off += kChunk, ++k) {
        const int b = int(k % kBuf);
        const size_t n = std::min(kChunk, bytes - off);
        if (used[b] && (e = cudaEventSynchronize(B.done[b])) != cudaSuccess)
            return e;
        par_memcpy(B.buf[b], static_cast<const char*>(host) + off, n);
        if ((e = cudaMemcpyAsync(static_cast<char*>(dev) + off, B.buf[b], n,
                                 cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return e;
        if ((e = cudaEventRecord(B.done[b], s)) != cudaSuccess)
            return e;
        used[b] = true;
    }
    return cudaStreamSynchronize(s);
}

cudaError_t d2h_large(void* host, const void* dev, size_t bytes, cudaStream_t s) {
    if (bytes < kDirect) {
        cudaError_t e = cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, s);
        return e != cudaSuccess ? e : cudaStreamSynchronize(s);
    }
    Bounce& B = t_bounce;
    cudaError_t e = B.ensure();
    if (e != cudaSuccess)
        return e;
    const size_t chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) -> cudaError_t {
        const size_t off = k * kChunk, n = std::min(kChunk, bytes - off);
        const int b = int(k % kBuf);
        cudaError_t r = cudaMemcpyAsync(B.buf[b], static_cast<const char*>(dev) + off, n,
                                        cudaMemcpyDeviceToHost, s);
        return r != cudaSuccess ? r : cudaEventRecord(B.done[b], s);
    };
    for (size_t k = 0; k + 1 < size_t(kBuf) && k < chunks; ++k)
        if ((e = issue(k)) != cudaSuccess)
            return e;
    for (size_t k = 0; k < chunks; ++k) {
        const int b = int(k % kBuf);
        if ((e = cudaEventSynchronize(B.done[b])) != cudaSuccess)
            return e;
        // the buffer drained last iteration is free again: keep kBuf - 1 DMAs queued
        if (k + kBuf - 1 < chunks && (e = issue(k + kBuf - 1)) != cudaSuccess)
            return e;
        const size_t off = k * kChunk, n = std::min(kChunk, bytes - off);
        par_memcpy(static_cast<char*>(host) + off, B.buf[b], n);
    }
    return cudaSuccess;
}

// ---- device block cache ------------------------------------------------------

namespace {

struct BlockCache {
    std::mutex mu;
    // (device, bytes) -> free blocks
    std::map<std::pair<int, size_t>, std::vector<void*>> free;
    size_t cached = 0;
    size_t limit = 0;
    bool enabled = true;
    BlockCache() {
        if (const char* e = std::getenv("PD_NO_BLOCK_CACHE"))
            enabled = std::atoi(e) == 0;
    }
};

BlockCache& cache() {
    static BlockCache* c = new BlockCache;  // never destroyed: blocks outlive static teardown
    return *c;
}

// every block is cached, small ones included: a cudaFree synchronises the
// device and was measured at up to 200 ms for a 24-byte block at the end of a
// 10M-node simulate() (PD_TIMING reports slow frees)
constexpr size_t kMinCached = 1;

} // namespace

cudaError_t dev_alloc(void** p, size_t bytes) {
    BlockCache& c = cache();
    int dev = 0;
    cudaGetDevice(&dev);
    if (c.enabled && bytes >= kMinCached) {
        std::lock_guard<std::mutex> lk(c.mu);
        auto it = c.free.find({dev, bytes});
        if (it != c.free.end() && !it->second.empty()) {
            *p = it->second.back();
            it->second.pop_back();
            c.cached -= bytes;
            return cudaSuccess;
        }
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation && c.enabled) {
        // give the cached blocks back and retry once
        cudaGetLastError();
        release_cached_blocks();
        e = cudaMalloc(p, bytes);
    }
    return e;
}

namespace {
// PD_TIMING: report device frees that take longer than 5 ms
struct SlowFree {
    bool on = std::getenv("PD_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    size_t bytes;
    const char* how = "cache";
    explicit SlowFree(size_t b) : bytes(b) {}
    ~SlowFree() {
        const double ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        if (on && ms > 5.0)
            std::fprintf(stderr, "[pd timing] dev_free %zu bytes (%s) %.3f ms\n", bytes, how, ms);
    }
};
} // namespace

void dev_free(void* p, size_t bytes) {
    BlockCache& c = cache();
    SlowFree sf(bytes);
    if (!c.enabled || bytes < kMinCached) {
        sf.how = "cudaFree";
        cudaFree(p);
        return;
    }
    int dev = 0;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) == cudaSuccess)
        dev = attr.device;
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.limit == 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        c.limit = tot / 2;  // keep at most half the device mapped for reuse
    }
    if (c.cached + bytes > c.limit) {
        sf.how = "cudaFree over limit";
        cudaFree(p);
        return;
    }
    c.free[{dev, bytes}].push_back(p);
    c.cached += bytes;
}

void release_cached_blocks() {
    BlockCache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    for (auto& kv : c.free)
        for (void* p : kv.second)
            cudaFree(p);
    c.free.clear();
    c.cached = 0;
}

} // namespace pdb

extern "C" void pd_release_cached_memory(void) { pdb::release_cached_blocks(); }
