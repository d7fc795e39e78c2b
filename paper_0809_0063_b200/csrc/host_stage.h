// Pinned staging of pageable host operands for the host pipeline (host_stage.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>

namespace qadic {

// slots [0, kStageIn): inputs (B chunks, then A panels); [kStageIn, 2 kStageIn): C panels.
// Three of each: the host copies C panel i-3 out while panels i-2..i are in flight,
// so it never waits on a transfer it has just queued.
constexpr int kStageIn = 3;
constexpr int kStageSlots = 2 * kStageIn;

// true for memory the driver does not know (malloc / numpy): neither device,
// managed nor page-locked
bool is_pageable(const void* p);

// memcpy split over a persistent pool of host threads
void parallel_copy(void* dst, const void* src, size_t bytes);

struct Ring;

// Exclusive use of the cached ring of pinned slots (each >= slot_bytes) for
// one host-pipeline call.  Slot i carries an event marking the last DMA that
// used it; the destructor waits for all of them.
class StageLease {
   public:
    explicit StageLease(size_t slot_bytes);
    ~StageLease();
    StageLease(const StageLease&) = delete;
    StageLease& operator=(const StageLease&) = delete;
    bool ok() const { return ok_; }
    uint8_t* slot(int i) const { return slot_[i]; }
    void wait(int i);                                // host waits until slot i is free
    void release_after(int i, cudaStream_t s);      // slot i busy until work queued on s so far completes
    // host -> slot i (parallel copy) -> device, on stream s
    void h2d(int i, void* dev, const void* host, size_t bytes, cudaStream_t s);

   private:
    Ring* ring_;
    std::lock_guard<std::mutex> lock_;
    uint8_t* slot_[kStageSlots] = {};
    bool ok_ = false;
};

}  // namespace qadic
