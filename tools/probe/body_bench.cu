// Cycle cost of one task-body call on a single CTA, data hot in L2/L1:
// through the device jump table (the worker's path), and the dense loop alone.
//   build/probe/body_bench
#include <cstdio>
#include <cstring>

#include "dev_common.cuh"
#include "dev_state.h"
#include "ops_elementwise.cuh"

namespace gdev {
__device__ __noinline__ int op_nop(const gpuos_task*, const Ctx*) { return 0; }
__device__ OpFn g_bench_fns[3] = {op_add, op_relu, op_nop};
}
using namespace gdev;

__global__ void __launch_bounds__(256, 1) body_bench(gpuos_task task, int reps, int mode, long long* cyc, int idle_ns) {
  __shared__ gpuos_task t;
  if (threadIdx.x == 0) t = task;
  __syncthreads();
  Ctx c;
  c.tid = threadIdx.x;
  c.nthreads = 256;
  c.part = 0;
  c.nparts = 1;
  c.bar_id = 1;
  c.smem = nullptr;
  c.smem_bytes = 0;
  c.aux = 0;
  c.flags = 0;
  c.tmem = kNoTmem;
  long long best = 1ll << 60, sum = 0;
  for (int r = 0; r < reps; ++r) {
    if (idle_ns) {
      // an idle gap like queue depth 1 (the host round trip between tasks)
      const unsigned long long g0 = globaltimer();
      while (globaltimer() - g0 < (unsigned long long)idle_ns) __nanosleep(1000);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const long long t0 = clock64();
    if (mode == 0) {
      g_bench_fns[0](&t, &c);
    } else if (mode == 2) {
      g_bench_fns[2](&t, &c);
    } else if (mode == 3) {
      ew_body<FAdd>(&t, &c, true);
    } else if (mode == 4) {
      c.flags = kPlanDenseSame;
      g_bench_fns[0](&t, &c);
    } else {
      FAdd f;
      ew_dense<GPUOS_F32>(&t, &c, t.views[0].extents[0], f);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const long long dt = clock64() - t0;
    if (r > 0) {
      sum += dt;
      best = dt < best ? dt : best;
    }
  }
  if (threadIdx.x == 0) {
    cyc[0] = best;
    cyc[1] = sum / (reps - 1);
  }
}

int main() {
  for (int n : {64, 4096, 65536}) {
    float *a, *b, *o;
    cudaMalloc(&a, n * 4);
    cudaMalloc(&b, n * 4);
    cudaMalloc(&o, n * 4);
    cudaMemset(a, 0, n * 4);
    cudaMemset(b, 0, n * 4);
    long long* cyc;
    cudaMallocManaged(&cyc, 16);
    gpuos_task t;
    std::memset(&t, 0, sizeof(t));
    t.op_id = 0;
    t.n_inputs = 2;
    t.size = n;
    float* ptrs[3] = {o, a, b};
    for (int v = 0; v < 3; ++v) {
      t.views[v].addr = (uint64_t)ptrs[v];
      t.views[v].rank = 1;
      t.views[v].extents[0] = n;
      t.views[v].strides[0] = 1;
      t.views[v].dtype = GPUOS_F32;
    }
    cudaDeviceSetLimit(cudaLimitStackSize, 4096);
    for (int idle : {0, 10000})
    for (int mode = 0; mode < 5; ++mode) {
      body_bench<<<1, 256>>>(t, 50, mode, cyc, idle);
      cudaError_t e = cudaDeviceSynchronize();
      std::printf("n=%6d idle=%5dns %-22s best %7lld cycles  mean %7lld cycles (%s)\n", n, idle,
                  mode == 0 ? "jump-table op_add" : mode == 1 ? "inline ew_dense<f32>" : mode == 2 ? "jump-table nop" : mode == 3 ? "inline ew_body<add>" : "jump-table op_add plan", cyc[0], cyc[1], cudaGetErrorString(e));
    }
  }
  return 0;
}
