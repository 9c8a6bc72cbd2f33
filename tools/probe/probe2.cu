// Second feasibility probe: on-device PCIe read latency of mapped pinned
// memory, host->device detection latency, cudaFree with a resident kernel,
// and module-load variants (EAGER env, cuLibraryLoadData, idle load time).
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>
#include <immintrin.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { std::printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); std::exit(1);} } while (0)

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ unsigned long long ld_sys(const volatile unsigned long long* p) { unsigned long long v; asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_sys(volatile unsigned long long* p, unsigned long long v) { asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }

struct Box { volatile unsigned long long cmd, resp, pad[6]; volatile unsigned long long data[64]; };

// (1) serial dependent reads of host memory, timed on device
__global__ void lat_kernel(Box* b, unsigned long long* out, int n) {
  unsigned long long acc = 0;
  for (int i = 0; i < n; ++i) {
    unsigned long long t0 = gt();
    acc += ld_sys(&b->data[(acc + i) & 7]);
    unsigned long long t1 = gt();
    out[i] = t1 - t0;
  }
  out[n] = acc;
}
// (1b) 384-byte warp-wide volatile read latency
__global__ void lat_warp_kernel(Box* b, unsigned long long* out, int n) {
  int lane = threadIdx.x;
  unsigned long long acc = 0;
  for (int i = 0; i < n; ++i) {
    unsigned long long t0 = gt();
    uint4 v = make_uint4(0,0,0,0);
    if (lane < 24) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x),"=r"(v.y),"=r"(v.z),"=r"(v.w) : "l"((const char*)b->data + 16*lane + (acc & 1)*0) : "memory");
    acc += __shfl_sync(0xffffffff, v.x, 0) + 1;
    unsigned long long t1 = gt();
    if (lane == 0) out[i] = t1 - t0;
  }
  if (lane == 0) out[n] = acc;
}
// (2) echo server: device polls cmd, answers resp; records detection stamps
__global__ void echo(Box* b, volatile int* stop) {
  if (blockIdx.x != 0) { while (*stop == 0) __nanosleep(2000); return; }
  if (threadIdx.x != 0) return;
  unsigned long long last = 0;
  for (;;) {
    unsigned long long c = ld_sys(&b->cmd);
    if (c == last) continue;
    last = c;
    if (c == ~0ull) { *stop = 1; st_sys(&b->resp, c); return; }
    st_sys(&b->resp, c);
  }
}

static Box* g_b; static int* g_stop; static cudaStream_t g_ks, g_side;
static void launch_echo() { CK(cudaMemsetAsync(g_stop, 0, 4, g_side)); CK(cudaStreamSynchronize(g_side)); g_b->resp = 0; g_b->cmd = 0; echo<<<148, 256, 0, g_ks>>>(g_b, g_stop); CK(cudaGetLastError()); }
static void stop_echo() { g_b->cmd = ~0ull; }
static bool guarded(const char* name, const std::function<void()>& fn) {
  std::atomic<bool> done{false};
  std::thread wd([&] { for (int i = 0; i < 200 && !done.load(); ++i) std::this_thread::sleep_for(std::chrono::milliseconds(10)); if (!done.load()) stop_echo(); });
  auto t0 = std::chrono::steady_clock::now(); fn();
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  done = true; wd.join();
  bool alive = cudaStreamQuery(g_ks) == cudaErrorNotReady;
  std::printf("%-40s %9.3f ms  %s\n", name, ms, alive ? "OK (kernel resident)" : "BLOCKED until kernel exit");
  if (!alive) { CK(cudaStreamSynchronize(g_ks)); launch_echo(); }
  return alive;
}
static const char* kSrc = "extern \"C\" __global__ void jk(int* p) { *p = 42; }\n";
static std::vector<char> cubin() {
  nvrtcProgram prog; nvrtcCreateProgram(&prog, kSrc, "j.cu", 0, nullptr, nullptr);
  const char* opts[] = {"-arch=sm_100a"};
  if (nvrtcCompileProgram(prog, 1, opts) != NVRTC_SUCCESS) std::exit(3);
  size_t n; nvrtcGetCUBINSize(prog, &n); std::vector<char> c(n); nvrtcGetCUBIN(prog, c.data()); nvrtcDestroyProgram(&prog); return c;
}
static double pct(std::vector<double> v, double p) { std::sort(v.begin(), v.end()); return v[(size_t)(p * (v.size() - 1))]; }

int main(int argc, char** argv) {
  CK(cudaSetDevice(0)); cuInit(0);
  CK(cudaStreamCreateWithFlags(&g_ks, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&g_side, cudaStreamNonBlocking));
  CK(cudaHostAlloc(&g_b, sizeof(Box), cudaHostAllocMapped)); std::memset((void*)g_b, 0, sizeof(Box));
  CK(cudaMalloc(&g_stop, 4));
  unsigned long long* d_out; CK(cudaMalloc(&d_out, 8 * 4097));
  std::vector<unsigned long long> h(4097);
  const char* env = std::getenv("CUDA_MODULE_LOADING");
  std::printf("CUDA_MODULE_LOADING=%s\n", env ? env : "(unset)");
  // (1)
  lat_kernel<<<1, 1, 0, g_side>>>(g_b, d_out, 4096); CK(cudaStreamSynchronize(g_side));
  CK(cudaMemcpy(h.data(), d_out, 8 * 4097, cudaMemcpyDeviceToHost));
  { std::vector<double> v(h.begin() + 16, h.begin() + 4096); std::printf("device ld.sys 8B host read latency: p50 %.0f ns p99 %.0f ns min %.0f\n", pct(v, .5), pct(v, .99), pct(v, 0)); }
  lat_warp_kernel<<<1, 32, 0, g_side>>>(g_b, d_out, 4096); CK(cudaStreamSynchronize(g_side));
  CK(cudaMemcpy(h.data(), d_out, 8 * 4097, cudaMemcpyDeviceToHost));
  { std::vector<double> v(h.begin() + 16, h.begin() + 4096); std::printf("device 384B warp host read latency: p50 %.0f ns p99 %.0f ns min %.0f\n", pct(v, .5), pct(v, .99), pct(v, 0)); }
  // (2) echo RTT
  launch_echo();
  { std::vector<double> lat; unsigned long long s = 0;
    for (int i = 0; i < 20000; ++i) { ++s; auto t0 = std::chrono::steady_clock::now(); g_b->cmd = s; while (g_b->resp != s) _mm_pause(); lat.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count()); }
    std::printf("echo RTT host->dev->host: p50 %.3f us p99 %.3f us min %.3f\n", pct(lat, .5), pct(lat, .99), pct(lat, 0)); }
  // (3) frees
  void* p = nullptr; CK(cudaMalloc(&p, 1 << 20));
  guarded("cudaFree device 1MB", [&] { CK(cudaFree(p)); });
  void* pm = nullptr; CK(cudaMallocManaged(&pm, 1 << 20));
  guarded("cudaFree managed 1MB", [&] { CK(cudaFree(pm)); });
  void* ph = nullptr; CK(cudaHostAlloc(&ph, 1 << 20, 0));
  guarded("cudaFreeHost 1MB", [&] { CK(cudaFreeHost(ph)); });
  guarded("cudaMalloc 256MB", [&] { CK(cudaMalloc(&p, 256 << 20)); });
  // (4) module load variants
  std::vector<char> cb = cubin();
  CUmodule mod; CUlibrary lib;
  guarded("cuModuleLoadData (resident kernel)", [&] { cuModuleLoadData(&mod, cb.data()); });
  guarded("cuLibraryLoadData (resident kernel)", [&] { CUresult r = cuLibraryLoadData(&lib, cb.data(), nullptr, nullptr, 0, nullptr, nullptr, 0); if (r) std::printf("lib err %d\n", r); });
  CUkernel kern;
  guarded("cuLibraryGetKernel", [&] { CUresult r = cuLibraryGetKernel(&kern, lib, "jk"); if (r) std::printf("getkernel err %d\n", r); });
  CUfunction f;
  guarded("cuKernelGetFunction", [&] { CUresult r = cuKernelGetFunction(&f, kern); if (r) std::printf("getfunc err %d\n", r); });
  stop_echo(); CK(cudaStreamSynchronize(g_ks));
  { auto t0 = std::chrono::steady_clock::now(); CUmodule m2; cuModuleLoadData(&m2, cb.data()); std::printf("cuModuleLoadData idle: %.3f ms\n", std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count()); }
  std::printf("probe2 done\n");
  return 0;
}
