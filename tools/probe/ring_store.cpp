// Host store strategies for ring slots in mapped pinned memory (no device).
//   build/probe/ring_store
#include <cuda_runtime.h>
#include <immintrin.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

static double now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static inline uint64_t mix(uint64_t w, uint32_t i) {
  uint64_t x = w + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull;
  x ^= x >> 31;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 29;
  return x;
}

int main() {
  const int cap = 16384, n = 200000;
  for (int slot : {384, 128}) {
    char* ring = nullptr;
    uint64_t* tail = nullptr;
    if (cudaHostAlloc((void**)&ring, (size_t)cap * slot, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostAlloc((void**)&tail, 4096, cudaHostAllocMapped) != cudaSuccess) {
      std::printf("(no GPU: plain host memory)\n");
      ring = (char*)aligned_alloc(4096, (size_t)cap * slot);
      tail = (uint64_t*)aligned_alloc(4096, 4096);
    }
    std::memset(ring, 0, (size_t)cap * slot);
    alignas(64) uint64_t w[48];
    for (int i = 0; i < 48; ++i) w[i] = i * 12345;
    const int words = slot / 8;
    for (int mode = 0; mode < 6; ++mode) {
      double t0 = now_ns();
      for (int k = 0; k < n; ++k) {
        char* dst = ring + (size_t)(k & (cap - 1)) * slot;
        w[0] = k + 1;
        if (mode == 0 || mode == 1 || mode == 4) {
          uint64_t h = 0;
          for (int i = 0; i < words; ++i)
            if (i != 7) h += mix(w[i], i);
          w[7] = h;
        }
        if (mode == 0 || mode == 2) {  // NT + sfence
          for (int i = 0; i < slot / 16; ++i)
            _mm_stream_si128((__m128i*)(dst + 16 * i), _mm_load_si128((const __m128i*)((const char*)w + 16 * i)));
          _mm_stream_si64((long long*)tail, k + 1);
          _mm_sfence();
        } else if (mode == 1 || mode == 3) {  // regular stores, release pub
          std::memcpy(dst + 8, (const char*)w + 8, slot - 8);
          __atomic_store_n((uint64_t*)dst, w[0], __ATOMIC_RELEASE);
          __atomic_store_n(tail, (uint64_t)k + 1, __ATOMIC_RELEASE);
        } else if (mode == 4) {  // NT, no fence, regular tail
          for (int i = 0; i < slot / 16; ++i)
            _mm_stream_si128((__m128i*)(dst + 16 * i), _mm_load_si128((const __m128i*)((const char*)w + 16 * i)));
          __atomic_store_n(tail, (uint64_t)k + 1, __ATOMIC_RELEASE);
        } else {  // AVX-512/256 regular
          for (int i = 0; i < slot / 32; ++i)
            _mm256_store_si256((__m256i*)(dst + 32 * i), _mm256_load_si256((const __m256i*)((const char*)w + 32 * i)));
          __atomic_store_n(tail, (uint64_t)k + 1, __ATOMIC_RELEASE);
        }
      }
      double t1 = now_ns();
      static const char* names[] = {"NT+sfence+chk", "regular+chk", "NT+sfence", "regular", "NT nofence+chk",
                                    "avx regular"};
      std::printf("slot %d %-16s %.1f ns/slot\n", slot, names[mode], (t1 - t0) / n);
    }
  }
  return 0;
}
