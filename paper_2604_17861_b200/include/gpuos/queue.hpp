// Task ring, host side (reference queue.hpp:156-300 restated over the C-ABI).
//
// The ring is the mapped-pinned array of 128-byte slots owned by
// libgpuos_cuda.so (include/gpuos_ring_format.h): the producer reserves a
// position, writes the slot (compact encoding, or slot + 256-byte extension
// record) and publishes it with word 0 = pos + 1; the persistent worker
// kernel is the consumer -- its fetcher warp claims tickets with an HBM
// atomic, reads the slot over PCIe and frees it (word 0 = pos + capacity).
// So the reference's producer half (acquire_slot / commit / peek / capacity)
// lives here, and its consumer half (try_claim / mark_done, executor.hpp
// worker_main) runs on the device (paper_2604_17861_b200/csrc/worker.cu).
// Runtime uses these calls through its own submit path; TaskQueue is the same
// producer API for callers that build gpuos_task descriptors themselves.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>

#include "gpuos_cuda.h"

namespace gpuos {

inline constexpr uint16_t kFlagFusedComposite = GPUOS_FLAG_FUSED_COMPOSITE;
inline constexpr uint16_t kFlagShutdown = GPUOS_FLAG_SHUTDOWN;
inline constexpr size_t kMaxInputs = GPUOS_MAX_INPUTS;
inline constexpr size_t kMaxScalars = GPUOS_MAX_SCALARS;
inline constexpr size_t kInlineRank = GPUOS_MAX_RANK;

class TaskQueue {
 public:
  struct Snapshot {
    uint64_t head = 0;       // tasks claimed by workers
    uint64_t tail = 0;       // tasks published
    uint64_t processed = 0;  // tasks completed
  };

  /// A view of the ring of an open device (single producer, queue.hpp:156-160).
  explicit TaskQueue(gpuos_dev* dev) : dev_(dev) {}

  /// Power-of-two slot count (queue.hpp:162-174).
  size_t capacity() const {
    uint64_t c = 0;
    gpuos_ring_capacity(dev_, &c);
    return static_cast<size_t>(c);
  }
  /// The next position, or nullopt when its slot is still owned by the
  /// previous lap (queue.hpp:179-190: full ring).
  std::optional<uint64_t> acquire_slot() {
    uint64_t pos = 0;
    if (gpuos_ring_reserve(dev_, &pos) != GPUOS_OK) return std::nullopt;
    return pos;
  }
  /// Encode and publish a descriptor at a reserved position (queue.hpp:192-231:
  /// inline views or the spill record, checksum, publication word last).
  void commit(uint64_t pos, const gpuos_task& task) { gpuos_ring_publish(dev_, pos, &task); }
  /// processed <= head <= tail at every instant (queue.hpp:272-279).
  Snapshot peek() const {
    gpuos_snapshot s{};
    gpuos_ring_peek(dev_, &s);
    Snapshot out;
    out.head = s.head;
    out.tail = s.tail;
    out.processed = s.processed;
    return out;
  }
  /// Block until the device processed count reaches `count` (queue.hpp:295-300).
  int wait_for_processed(uint64_t count) { return gpuos_ring_wait_processed(dev_, count); }

 private:
  gpuos_dev* dev_;
};

}  // namespace gpuos
