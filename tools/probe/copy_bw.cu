// PCIe copy bandwidth on the box: pinned H2D, D2H, and both at once.
#include <cuda_runtime.h>
#include <cstdio>
int main() {
  const size_t a = 327680000, b = 163840000;
  void *ha, *hb, *da, *db;
  cudaHostAlloc(&ha, a, cudaHostAllocPortable);
  cudaHostAlloc(&hb, b, cudaHostAllocPortable);
  cudaMalloc(&da, a);
  cudaMalloc(&db, b);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int r = 0; r < 3; ++r) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      if (mode != 1) cudaMemcpyAsync(da, ha, a, cudaMemcpyHostToDevice, s1);
      if (mode != 0) cudaMemcpyAsync(hb, db, b, cudaMemcpyDeviceToHost, s2);
      cudaDeviceSynchronize();
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* nm[] = {"H2D 327.7MB", "D2H 163.8MB", "both"};
      std::printf("%-12s %.3f ms  (%.1f GB/s total)\n", nm[mode], ms,
                  ((mode != 1 ? a : 0) + (mode != 0 ? b : 0)) / (ms * 1e6));
    }
  return 0;
}
