// Ring wire format shared by the host publisher (capi.cu) and the device
// fetcher (worker.cu).  Replaces PackedDescriptor (reference queue.hpp:62-142).
//
// A ring slot is 128 bytes (one warp-wide read covers four slots).  The ABI
// descriptor (gpuos_task, 384 B) travels in one of two encodings:
//
//   compact (kFmtCompact): every operand view -- output and n_inputs inputs --
//     bound cleanly, has the output's dtype and rank/extents and row-major
//     contiguous strides, and at most one scalar is set.  The small-op common
//     case.  16 words:
//       w0 publication word     w1 seq
//       w2 op_id | flags<<32 | n_inputs<<48 | n_scalars<<56
//       w3 size                 w4 done_cell          w5 enqueue stamp
//       w6 fmt | dtype<<8 | rank<<16                  w7 checksum
//       w8..w9 extents[4] (int32)                     w10..w14 addr[5]
//       w15 scalars[0]
//
//   extended (kFmtExtended): anything else.  The slot holds gpuos_task words
//     0..15 (header + the 8 scalars; w6 = fmt), and the views -- task words
//     16..46 -- sit in a 256-byte extension record of the same ring index (the
//     reference's spill table, queue.hpp:207-221), with ext word 31 = its own
//     checksum bound to the ring position.  The host writes the record before
//     the slot; the fetcher reads it after the slot validated.
//
// Checksums: Σ w[i]·(2i+1) mod 2^64 over the other words (slot_term in
// dev_common.cuh); the extension adds slot_term(pos + 1, 40) so a record left
// from an earlier lap cannot validate.
#pragma once

#include <stdint.h>

#include "gpuos_cuda.h"

#ifdef __CUDACC__
#define GPUOS_RING_FN __host__ __device__ __forceinline__
#else  // host-only C++ (the runtime header writes dense slots inline)
#define GPUOS_RING_FN inline
#endif

namespace gdev {

constexpr uint32_t kRingSlot = 128;  // bytes per ring slot
constexpr uint32_t kExtBytes = 256;  // bytes per extension record
constexpr uint32_t kSlotWords = kRingSlot / 8;
constexpr uint32_t kExtWords = kExtBytes / 8;
constexpr uint32_t kFmtExtended = 0;
constexpr uint32_t kFmtCompact = 1;
constexpr uint32_t kExtChecksumSalt = 40;

GPUOS_RING_FN uint64_t ring_term(uint64_t w, uint32_t i) { return w * (uint64_t)(2 * i + 1); }

// Row-major contiguous strides of `rank` extents (unit dims included), the
// strides a compact view expands to.
GPUOS_RING_FN void contiguous_strides4(const int32_t* ext, int rank, int32_t* st) {
  int64_t s = 1;
  for (int d = 3; d >= 0; --d) {
    if (d >= rank) {
      st[d] = 0;
      continue;
    }
    st[d] = (int32_t)s;
    s *= ext[d];
  }
}

}  // namespace gdev
