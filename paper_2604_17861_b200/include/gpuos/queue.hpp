// Task-ring vocabulary shared with the reference API (queue.hpp:22-58,
// 156-160).  The ring itself is the mapped-pinned slot array managed by
// libgpuos_cuda.so (gpuos_ring_*): 384-byte slots with a per-slot lap
// sequence word, consumed by the persistent worker kernel over PCIe.
#pragma once

#include <cstddef>
#include <cstdint>

#include "gpuos_cuda.h"

namespace gpuos {

inline constexpr uint16_t kFlagFusedComposite = GPUOS_FLAG_FUSED_COMPOSITE;
inline constexpr uint16_t kFlagShutdown = GPUOS_FLAG_SHUTDOWN;
inline constexpr size_t kMaxInputs = GPUOS_MAX_INPUTS;
inline constexpr size_t kMaxScalars = GPUOS_MAX_SCALARS;
inline constexpr size_t kInlineRank = GPUOS_MAX_RANK;

struct TaskQueue {
  struct Snapshot {
    uint64_t head = 0;       // tasks claimed by workers
    uint64_t tail = 0;       // tasks published
    uint64_t processed = 0;  // tasks completed
  };
};

}  // namespace gpuos
