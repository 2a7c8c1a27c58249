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

struct Bounce {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int device = -1;
    ~Bounce() {
        for (int k = 0; k < 2; ++k) {
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
        for (int k = 0; k < 2; ++k) {
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

// memcpy split over a few host threads (one memcpy stream tops out near
// 10 GB/s; the chunk is large enough to amortise the thread start)
void par_memcpy(void* dst, const void* src, size_t bytes) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t parts = std::min<size_t>({size_t(8), size_t(hw), bytes / (size_t(4) << 20) + 1});
    if (parts <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    const size_t step = (bytes + parts - 1) / parts;
    for (size_t p = 0; p < parts; ++p) {
        const size_t b = p * step, e = std::min(bytes, b + step);
        if (b < e)
            th.emplace_back([=] {
                std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b);
            });
    }
    for (auto& t : th)
        t.join();
}

} // namespace

cudaError_t h2d_large(void* dev, const void* host, size_t bytes, cudaStream_t s) {
    if (bytes < kDirect)
        return cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, s);
    Bounce& B = t_bounce;
    cudaError_t e = B.ensure();
    if (e != cudaSuccess)
        return e;
    bool used[2] = {false, false};
    for (size_t off = 0, k = 0; off < bytes; off += kChunk, ++k) {
        const int b = int(k & 1);
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
        const int b = int(k & 1);
        cudaError_t r = cudaMemcpyAsync(B.buf[b], static_cast<const char*>(dev) + off, n,
                                        cudaMemcpyDeviceToHost, s);
        return r != cudaSuccess ? r : cudaEventRecord(B.done[b], s);
    };
    if ((e = issue(0)) != cudaSuccess)
        return e;
    for (size_t k = 0; k < chunks; ++k) {
        const int b = int(k & 1);
        if ((e = cudaEventSynchronize(B.done[b])) != cudaSuccess)
            return e;
        if (k + 1 < chunks && (e = issue(k + 1)) != cudaSuccess)
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

// blocks below 1 MB are not worth caching
constexpr size_t kMinCached = size_t(1) << 20;

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

void dev_free(void* p, size_t bytes) {
    BlockCache& c = cache();
    if (!c.enabled || bytes < kMinCached) {
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
