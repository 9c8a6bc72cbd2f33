// Cycle cost of single task bodies (one CTA, 128-thread group like the
// worker's executor groups, data hot in L2): softmax 128x128, mul by a rank-0
// scalar 128x64, for bf16 and f32.
#include <cstdio>
#include <cstring>

#include "dev_common.cuh"
#include "dev_state.h"
#include "ops_elementwise.cuh"
#include "ops_linalg.cuh"
#include "ops_rowwise.cuh"

namespace gdev {
__device__ OpFn g_b2_fns[2] = {op_softmax, op_mul};
}
using namespace gdev;

__global__ void __launch_bounds__(128, 1) body_bench2(gpuos_task task, int which, int reps, long long* cyc) {
  __shared__ gpuos_task t;
  extern __shared__ char scratch[];
  if (threadIdx.x == 0) t = task;
  __syncthreads();
  Ctx c;
  c.tid = threadIdx.x;
  c.nthreads = 128;
  c.part = 0;
  c.nparts = 1;
  c.bar_id = 1;
  c.smem = scratch;
  c.smem_bytes = 32768;
  c.aux = 0;
  c.flags = 0;
  c.tmem = kNoTmem;
  long long best = 1ll << 60;
  for (int r = 0; r < reps; ++r) {
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const long long t0 = clock64();
    int rc = g_b2_fns[which](&t, &c);
    asm volatile("bar.sync 1, 128;" ::: "memory");
    const long long dt = clock64() - t0;
    if (r > 0 && dt < best) best = dt;
    if (rc && threadIdx.x == 0) cyc[1] = rc;
  }
  if (threadIdx.x == 0) cyc[0] = best;
}

int main() {
  for (int dt : {GPUOS_F32, GPUOS_BF16}) {
    const int w = dt == GPUOS_F32 ? 4 : 2;
    void *a, *b, *o;
    cudaMalloc(&a, 128 * 128 * 4);
    cudaMalloc(&b, 16);
    cudaMalloc(&o, 128 * 128 * 4);
    cudaMemset(a, 0, 128 * 128 * 4);
    cudaMemset(b, 0, 16);
    long long* cyc;
    cudaMallocManaged(&cyc, 16);
    for (int which = 0; which < 2; ++which) {
      gpuos_task t;
      std::memset(&t, 0, sizeof(t));
      int rows = 128, cols = which == 0 ? 128 : 64;
      t.n_inputs = which == 0 ? 1 : 2;
      t.views[0].addr = (uint64_t)o;
      t.views[1].addr = (uint64_t)a;
      t.views[2].addr = (uint64_t)b;
      for (int v = 0; v < 2; ++v) {
        t.views[v].rank = 2;
        t.views[v].extents[0] = rows;
        t.views[v].extents[1] = cols;
        t.views[v].strides[0] = cols;
        t.views[v].strides[1] = 1;
        t.views[v].dtype = dt;
      }
      t.views[2].rank = 0;
      t.views[2].dtype = dt;
      cyc[1] = 0;
      cudaFuncSetAttribute(body_bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
      body_bench2<<<1, 128, 32768>>>(t, which, 20, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      std::printf("dtype %d %-8s best %8lld cycles = %.2f us (rc %lld, %s)\n", dt, which == 0 ? "softmax" : "mul-rank0",
                  cyc[0], cyc[0] / 1965.0, cyc[1], cudaGetErrorString(e));
    }
    (void)w;
  }
  return 0;
}
