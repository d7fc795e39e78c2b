// Host-side staging for pageable (unregistered) operands of the host pipeline.
//
// A DMA from pageable memory runs through the driver's own small bounce
// buffers, synchronously and at a fraction of the PCIe rate (cfg5 numpy in /
// numpy out: 46.7 ms against 8.8 ms from pinned buffers).  Instead the
// pipeline copies each panel into a page-locked slot with a pool of host
// threads (~47 GB/s on the 16-core host, close to the PCIe rate) while the
// device works on the previous panel, and DMAs from the slot.  Results come back the same way:
// D2H into a pinned slot, then a parallel copy into the caller's buffer.
//
// Pieces: a persistent copy pool (one job at a time, split into page-aligned
// parts, the calling thread takes part 0) and a cached ring of pinned slots
// guarded by a mutex (a staged call owns the ring until it returns).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "host_stage.h"

namespace qadic {

namespace {

class CopyPool {
   public:
    explicit CopyPool(int workers) {
        for (int t = 0; t < workers; ++t) threads_.emplace_back([this, t] { loop(t + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& th : threads_) th.join();
    }
    int parts() const { return (int)threads_.size() + 1; }

    void copy(void* dst, const void* src, size_t bytes) {
        if (bytes == 0) return;
        const size_t min_part = size_t(1) << 20;
        int np = (int)std::min<size_t>((size_t)parts(), (bytes + min_part - 1) / min_part);
        if (np <= 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> g(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            np_ = np;
            pending_ = np - 1;
            ++gen_;
        }
        cv_.notify_all();
        run_part(0);
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return pending_ == 0; });
    }

   private:
    void run_part(int i) {
        // page-aligned parts: workers never share a page
        const size_t per = ((bytes_ + np_ - 1) / np_ + 4095) & ~size_t(4095);
        const size_t b0 = std::min(bytes_, per * (size_t)i), b1 = std::min(bytes_, b0 + per);
        if (b1 > b0) std::memcpy(dst_ + b0, src_ + b0, b1 - b0);
    }
    void loop(int idx) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> g(mu_);
            cv_.wait(g, [&] { return gen_ != seen; });
            seen = gen_;
            if (stop_) return;
            if (idx >= np_) continue;
            g.unlock();
            run_part(idx);
            g.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }

    std::vector<std::thread> threads_;
    std::mutex mu_, job_mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int np_ = 0, pending_ = 0;
};

int pool_workers() {
    const char* e = std::getenv("QADIC_COPY_THREADS");
    // default: half the hardware threads, at most 8 -- the copies are bound by host
    // memory bandwidth shared with the DMA engines (8 measured >= 12 or 16 at cfg5)
    int n = e ? std::atoi(e) : std::min(8, std::max(1, (int)std::thread::hardware_concurrency() / 2));
    return std::max(1, std::min(n, 64)) - 1;  // the caller is one of the copiers
}

}  // namespace

struct Ring {
    std::mutex mu;
    uint8_t* base = nullptr;
    size_t slot_bytes = 0;
    cudaEvent_t ev[kStageSlots] = {};
};

namespace {

Ring& ring() {  // one ring per device (its events belong to that device)
    static Ring r[64];
    int dev = 0;
    cudaGetDevice(&dev);
    return r[dev & 63];
}

}  // namespace

void parallel_copy(void* dst, const void* src, size_t bytes) {
    static CopyPool pool(pool_workers());
    pool.copy(dst, src, bytes);
}

bool is_pageable(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
}

StageLease::StageLease(size_t slot_bytes) : ring_(&ring()), lock_(ring_->mu) {
    Ring& r = *ring_;
    slot_bytes = (slot_bytes + 4095) & ~size_t(4095);
    if (r.slot_bytes < slot_bytes) {
        if (r.base) cudaFreeHost(r.base);
        r.base = nullptr;
        r.slot_bytes = 0;
        if (cudaHostAlloc(reinterpret_cast<void**>(&r.base), slot_bytes * kStageSlots, cudaHostAllocPortable) !=
            cudaSuccess) {
            cudaGetLastError();
            r.base = nullptr;
            return;
        }
        r.slot_bytes = slot_bytes;
    }
    for (int i = 0; i < kStageSlots; ++i) {
        if (!r.ev[i]) cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming | cudaEventBlockingSync);
        slot_[i] = r.base + (size_t)i * r.slot_bytes;
    }
    ok_ = true;
}

StageLease::~StageLease() {
    // every DMA that reads or writes a slot has completed before the ring is released
    if (ok_)
        for (int i = 0; i < kStageSlots; ++i) cudaEventSynchronize(ring_->ev[i]);
}

void StageLease::wait(int i) { cudaEventSynchronize(ring_->ev[i]); }
void StageLease::release_after(int i, cudaStream_t s) { cudaEventRecord(ring_->ev[i], s); }

void StageLease::h2d(int i, void* dev, const void* host, size_t bytes, cudaStream_t s) {
    wait(i);
    parallel_copy(slot_[i], host, bytes);
    cudaMemcpyAsync(dev, slot_[i], bytes, cudaMemcpyHostToDevice, s);
    release_after(i, s);
}

}  // namespace qadic
