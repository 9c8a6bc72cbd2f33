// PCIe round-trip floor for the submit->complete path: one GPU thread polls a
// word in mapped pinned memory and answers in another; the host times
// write->answer.  Mode 0: relaxed.sys loads/stores.  Mode 1: the answer is
// preceded by fence.release.gpu (what a completer pays).  Mode 2: the poller
// also reads a 128-byte slot (one warp, v4 per lane) like the fetcher.  Mode 3:
// the fetcher's full round (slot + host tail + device control words).  Mode 4:
// mode 3 without the host-tail read.
#include <cuda_runtime.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

__global__ void pong(volatile uint64_t* flag, volatile uint64_t* ack, const uint4* slot, int iters, int mode,
                     const uint64_t* dev) {
  const int lane = threadIdx.x;
  uint64_t acc = 0;
  for (int i = 1; i <= iters; ++i) {
    uint64_t v;
    do {
      if (mode >= 3) {
        // the fetcher's round: slot + control words (device, gpu scope) + the
        // host tail (sys) on single lanes, all issued before any is consumed
        uint4 s = make_uint4(0, 0, 0, 0);
        uint64_t aux = 0;
        if (lane < 8) asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s.x), "=r"(s.y), "=r"(s.z), "=r"(s.w) : "l"(slot + lane) : "memory");
        if (mode == 3 && lane == 4) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(aux) : "l"(flag + 8) : "memory");
        if (lane >= 1 && lane <= 6 && lane != 4) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(aux) : "l"(dev + lane * 16) : "memory");
        acc += __shfl_sync(0xffffffffu, aux, 5);
        v = __shfl_sync(0xffffffffu, ((uint64_t)s.y << 32) | s.x, 0);
      } else if (mode == 2) {
        uint4 s;
        asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(s.x), "=r"(s.y), "=r"(s.z), "=r"(s.w) : "l"(slot + (lane & 7)) : "memory");
        v = __shfl_sync(0xffffffffu, ((uint64_t)s.y << 32) | s.x, 0);
      } else {
        asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
        v = __shfl_sync(0xffffffffu, v, 0);
      }
    } while (v != (uint64_t)i);
    if (lane == 0) {
      if (mode >= 1) asm volatile("fence.release.gpu;" ::: "memory");
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(ack), "l"((uint64_t)i + (acc & 0)) : "memory");
    }
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 2000;
  uint64_t* devbuf;
  cudaMalloc(&devbuf, 4096);
  cudaMemset(devbuf, 0, 4096);
  for (int mode = 0; mode < 5; ++mode) {
    uint64_t* h;
    cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
    std::fill(h, h + 512, 0);
    uint64_t* d;
    cudaHostGetDevicePointer(&d, h, 0);
    volatile uint64_t* flag = h;
    volatile uint64_t* ack = h + 64;
    uint64_t* slot = h + 128;  // 128-byte slot; word 0 is the publication word
    pong<<<1, 32>>>((volatile uint64_t*)d, (volatile uint64_t*)(d + 64), (const uint4*)(d + 128), iters, mode, devbuf);
    std::vector<double> lat;
    for (int i = 1; i <= iters; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      if (mode >= 2) __atomic_store_n(slot, (uint64_t)i, __ATOMIC_RELEASE);
      else __atomic_store_n(flag, (uint64_t)i, __ATOMIC_RELEASE);
      while (*ack != (uint64_t)i) {
      }
      auto t1 = std::chrono::steady_clock::now();
      lat.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    cudaDeviceSynchronize();
    std::sort(lat.begin() + 100, lat.end());
    const size_t m = lat.size() - 100;
    printf("mode %d: p50 %.2f us p90 %.2f us p99 %.2f us\n", mode, lat[100 + m / 2], lat[100 + m * 9 / 10], lat[100 + m * 99 / 100]);
    cudaFreeHost(h);
  }
  return 0;
}
