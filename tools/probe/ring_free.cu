// Producer slot-write cost vs how the device frees ring slots (probe only).
//   build/probe/ring_free
// A host thread publishes 128-byte slots (15 words + checksum + publication
// word, then the tail) into a 4096-slot mapped ring, while 148 device CTAs
// claim tickets with an HBM atomic, poll their slot over PCIe and free it:
//   mode 0: free by writing the slot's word 0 = pos + cap (the round-1 protocol;
//           the host line is invalidated by the device write every lap)
//   mode 1: free by writing a 16-bit lap tag into a separate tag array (the
//           slot lines are only ever read by the device)
//   mode 2: free tags as mode 1, but the host checks a tag only once per 32
//           slots (one tag line) and prefetches the next tag line
// Prints host ns per published slot.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <x86intrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>

static double now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void consumer(const char* ring, uint16_t* tags, volatile uint64_t* tail, unsigned long long* claim,
                         uint64_t n, uint64_t cap, int mode) {
  if (threadIdx.x != 0) return;
  for (;;) {
    const uint64_t pos = atomicAdd(claim, 1ull);
    if (pos >= n) return;
    const uint64_t* slot = (const uint64_t*)(ring + (pos & (cap - 1)) * 128);
    uint64_t w0;
    do {
      asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w0) : "l"(slot) : "memory");
    } while (w0 != pos + 1);
    uint64_t w5;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w5) : "l"(slot + 5) : "memory");
    if (mode == 0) {
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(pos + cap) : "memory");
    } else {
      const uint16_t lap = (uint16_t)(pos / cap + 1);
      asm volatile("st.relaxed.sys.global.u16 [%0], %1;" ::"l"(tags + (pos & (cap - 1))), "h"(lap) : "memory");
    }
  }
}

int main() {
  const uint64_t cap = 4096, n = 400000;
  char* ring;
  uint16_t* tags;
  uint64_t* tail;
  cudaHostAlloc((void**)&ring, cap * 128, cudaHostAllocMapped);
  cudaHostAlloc((void**)&tags, cap * 2, cudaHostAllocMapped);
  cudaHostAlloc((void**)&tail, 4096, cudaHostAllocMapped);
  unsigned long long* claim;
  cudaMalloc(&claim, 8);
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      std::memset(ring, 0, cap * 128);
      std::memset(tags, 0, cap * 2);
      for (uint64_t i = 0; i < cap; ++i) *(uint64_t*)(ring + i * 128) = i;
      *tail = 0;
      cudaMemset(claim, 0, 8);
      cudaDeviceSynchronize();
      consumer<<<148, 32>>>(ring, tags, tail, claim, n, cap, mode);
      alignas(64) uint64_t w[16];
      for (int i = 0; i < 16; ++i) w[i] = i * 12345;
      uint64_t spins = 0;
      const double t0 = now_ns();
      for (uint64_t p = 0; p < n; ++p) {
        uint64_t* dst = (uint64_t*)(ring + (p & (cap - 1)) * 128);
        if (mode == 0) {
          while (__atomic_load_n(dst, __ATOMIC_ACQUIRE) != p) ++spins;
          __builtin_prefetch(ring + ((p + 16) & (cap - 1)) * 128, 1);
        } else if (mode == 1) {
          if (p >= cap) {
            const uint16_t want = (uint16_t)(p / cap);
            while (__atomic_load_n(&tags[p & (cap - 1)], __ATOMIC_ACQUIRE) != want) ++spins;
          }
        } else {
          if (p >= cap && (p & 31) == 0) {
            const uint16_t want = (uint16_t)(p / cap);
            // the whole 32-slot group must be free: check its last tag
            while (__atomic_load_n(&tags[(p + 31) & (cap - 1)], __ATOMIC_ACQUIRE) != want) ++spins;
            for (int k = 0; k < 32; ++k)
              while (__atomic_load_n(&tags[(p + k) & (cap - 1)], __ATOMIC_ACQUIRE) != want) ++spins;
            __builtin_prefetch(&tags[(p + 64) & (cap - 1)], 0);
          }
        }
        w[1] = p;
        uint64_t h = (p + 1);
        for (int i = 1; i < 16; ++i)
          if (i != 7) h += w[i] * (2 * i + 1);
        w[7] = h;
        for (int i = 1; i < 16; ++i) dst[i] = w[i];
        __atomic_store_n(&dst[0], p + 1, __ATOMIC_RELEASE);
        __atomic_store_n(tail, p + 1, __ATOMIC_RELEASE);
      }
      const double t1 = now_ns();
      cudaError_t e = cudaDeviceSynchronize();
      const double t2 = now_ns();
      std::printf("mode %d: host %.1f ns/slot (spins/slot %.2f), drain %.1f us, %s\n", mode, (t1 - t0) / n,
                  (double)spins / n, (t2 - t1) / 1e3, cudaGetErrorString(e));
    }
  return 0;
}
