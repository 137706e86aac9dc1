// Pageable host -> device staging (bind_input of plain numpy arrays, the reference Backend's
// std::vector operands).  cudaMemcpyAsync from pageable memory is staged by the driver on the
// calling thread (~10-12 GB/s measured on the box); here a pool of worker threads copies each
// 4 MiB slot of a pinned ring in parallel (host memcpy ~54 GB/s on eight threads,
// scripts/xfer_probe.py) while the previous slot's DMA runs, so the copy approaches the PCIe
// rate instead of the single-thread memcpy rate.
#include "hostcopy.hpp"

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <vector>

namespace spdzb200 {

namespace {

// Fixed worker pool: a copy job is split into (workers + 1) slices, the caller takes one.
class CopyPool {
public:
    explicit CopyPool(int workers) {
        for (int w = 0; w < workers; ++w) th_.emplace_back([this, w] { loop(w); });
    }
    ~CopyPool() {
        {
            std::lock_guard lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        const int parts = (int)th_.size() + 1;
        if (bytes < (1u << 20) || parts == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = (int)th_.size();
            ++gen_;
        }
        cv_.notify_all();
        slice(parts - 1, parts);  // the caller's own slice
        std::unique_lock lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

private:
    void slice(int k, int parts) {
        const size_t per = (bytes_ / parts + 63) & ~size_t(63);
        const size_t lo = std::min(bytes_, per * k), hi = k + 1 == parts ? bytes_ : std::min(bytes_, per * (k + 1));
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void loop(int w) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            slice(w, (int)th_.size() + 1);
            std::lock_guard lk(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    bool stop_ = false;
    int pending_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
};

constexpr size_t kSlot = 4u << 20;
constexpr int kSlots = 4;

struct Ring {  // per device: pinned slots and the event of each slot's last DMA
    char* slot[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
    bool used[kSlots] = {};
    int next = 0;
};

std::mutex g_mu;  // one staged copy at a time (the pool and the rings are shared)
std::map<int, Ring> g_rings;

CopyPool& pool() {
    static CopyPool p(std::max(1, std::min(7, (int)std::thread::hardware_concurrency() - 1)));
    return p;
}

}  // namespace

bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

namespace {
cudaError_t ring_ready(Ring& ring) {
    if (ring.slot[kSlots - 1] && ring.ev[kSlots - 1]) return cudaSuccess;
    for (int s = 0; s < kSlots; ++s) {
        cudaError_t e = cudaSuccess;
        if (!ring.slot[s]) {
            void* p = nullptr;
            e = cudaMallocHost(&p, kSlot);
            ring.slot[s] = e == cudaSuccess ? static_cast<char*>(p) : nullptr;
        }
        if (e == cudaSuccess && !ring.ev[s]) e = cudaEventCreateWithFlags(&ring.ev[s], cudaEventDisableTiming);
        if (e != cudaSuccess) {  // a later call retries the missing slots (a null slot is never used)
            if (ring.slot[s] && !ring.ev[s]) {
                cudaFreeHost(ring.slot[s]);
                ring.slot[s] = nullptr;
            }
            return e;
        }
    }
    return cudaSuccess;
}
}  // namespace

void parallel_copy(void* dst, const void* src, size_t bytes) {
    std::lock_guard lk(g_mu);
    pool().copy(dst, src, bytes);
}

cudaError_t staged_d2h(int device, void* host_dst, const void* src_dev, size_t bytes, cudaStream_t stream) {
    std::lock_guard lk(g_mu);
    Ring& ring = g_rings[device];
    cudaError_t e = ring_ready(ring);
    if (e != cudaSuccess) return e;
    for (int s = 0; s < kSlots; ++s)  // the ring's earlier H2D slots must be free
        if (ring.used[s] && (e = cudaEventSynchronize(ring.ev[s])) != cudaSuccess) return e;
    const char* src = static_cast<const char*>(src_dev);
    char* dst = static_cast<char*>(host_dst);
    const size_t chunks = (bytes + kSlot - 1) / kSlot;
    auto enqueue = [&](size_t c) {
        const size_t off = c * kSlot, n = std::min(kSlot, bytes - off);
        const int s = (int)(c % kSlots);
        cudaError_t r = cudaMemcpyAsync(ring.slot[s], src + off, n, cudaMemcpyDeviceToHost, stream);
        if (r == cudaSuccess) r = cudaEventRecord(ring.ev[s], stream);
        ring.used[s] = true;
        return r;
    };
    for (size_t c = 0; c < chunks && c < (size_t)kSlots; ++c)
        if ((e = enqueue(c)) != cudaSuccess) return e;
    for (size_t c = 0; c < chunks; ++c) {  // copy out slot c, then reuse it for chunk c + kSlots
        const int s = (int)(c % kSlots);
        if ((e = cudaEventSynchronize(ring.ev[s])) != cudaSuccess) return e;
        const size_t off = c * kSlot, n = std::min(kSlot, bytes - off);
        pool().copy(dst + off, ring.slot[s], n);
        if (c + kSlots < chunks && (e = enqueue(c + kSlots)) != cudaSuccess) return e;
    }
    ring.next = 0;
    return cudaSuccess;
}

cudaError_t staged_h2d(int device, void* dst_dev, const void* src_host, size_t bytes, cudaStream_t stream) {
    std::lock_guard lk(g_mu);
    Ring& ring = g_rings[device];
    if (cudaError_t e = ring_ready(ring); e != cudaSuccess) return e;
    const char* src = static_cast<const char*>(src_host);
    char* dst = static_cast<char*>(dst_dev);
    for (size_t off = 0; off < bytes; off += kSlot) {
        const size_t n = std::min(kSlot, bytes - off);
        const int s = ring.next;
        ring.next = (s + 1) % kSlots;
        if (ring.used[s]) {
            cudaError_t e = cudaEventSynchronize(ring.ev[s]);  // the slot's previous DMA is done
            if (e != cudaSuccess) return e;
        }
        pool().copy(ring.slot[s], src + off, n);
        cudaError_t e = cudaMemcpyAsync(dst + off, ring.slot[s], n, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = cudaEventRecord(ring.ev[s], stream);
        if (e != cudaSuccess) return e;
        ring.used[s] = true;
    }
    return cudaSuccess;
}

}  // namespace spdzb200
