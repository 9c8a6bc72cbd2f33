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

#if !defined(__CUDACC_RTC__)
// Compact-slot publisher (host): reserve, encode, checksum, publish word last,
// then the tail.  gpuos_ring_submit_dense and the runtime's inline dense path
// both run this.  x86 TSO orders the write-back stores for the device's
// coherent PCIe reads; a read interleaving with them fails the checksum.
// (Streaming stores, which skip the read-for-ownership, measured 4x slower:
// 210 vs 55 ns per task.)
inline int ring_write_dense(const gpuos_ring_view& r, const gpuos_dense_task& t) {
  const uint64_t p = *r.reserve;
  uint64_t* dst = reinterpret_cast<uint64_t*>(r.ring + (p & r.mask) * kRingSlot);
  if (__atomic_load_n(dst, __ATOMIC_ACQUIRE) != p) return GPUOS_QUEUE_FULL;
  *r.reserve = p + 1;
  // the device freed upcoming slots over PCIe (invalidating their first line
  // in the host caches): fetch one for writing well ahead of use
  __builtin_prefetch(r.ring + ((p + 16) & r.mask) * kRingSlot, 1);
  uint64_t w[kSlotWords];
  w[1] = t.seq;
  w[2] = (uint64_t)t.op_id | ((uint64_t)t.flags << 32) | ((uint64_t)t.n_inputs << 48) | ((uint64_t)t.n_scalars << 56);
  w[3] = t.size;
  w[4] = t.done_cell;
  w[5] = (t.flags & GPUOS_FLAG_AFTER) ? t.wait_target : (*r.trace_on ? __builtin_ia32_rdtsc() : 0);
  w[6] = kFmtCompact | ((uint64_t)t.dtype << 8) | ((uint64_t)t.rank << 16);
  w[8] = (uint64_t)(uint32_t)t.extents[0] | ((uint64_t)(uint32_t)t.extents[1] << 32);
  w[9] = (uint64_t)(uint32_t)t.extents[2] | ((uint64_t)(uint32_t)t.extents[3] << 32);
  for (int k = 0; k <= GPUOS_MAX_INPUTS; ++k) w[10 + k] = k <= t.n_inputs ? t.addr[k] : 0;
  __builtin_memcpy(&w[15], &t.scalar0, 8);
  uint64_t h = ring_term(p + 1, 0);
  for (uint32_t i = 1; i < kSlotWords; ++i)
    if (i != 7) h += ring_term(w[i], i);
  w[7] = h;
  for (uint32_t i = 1; i < kSlotWords; ++i) dst[i] = w[i];
  __atomic_store_n(&dst[0], p + 1, __ATOMIC_RELEASE);
  __atomic_store_n(r.tail, p + 1, __ATOMIC_RELEASE);
  return GPUOS_OK;
}
#endif

}  // namespace gdev
