// Feasibility probe for the persistent-kernel design (run once on a B200):
//  1. host->device->host ping-pong latency through mapped pinned memory
//  2. which CUDA APIs block while a persistent kernel is resident
//  3. NVRTC/nvJitLink -rdc cubin loaded into a live context, its device
//     function pointer called from the already-running kernel
// Every potentially-blocking call runs under a watchdog that releases the
// persistent kernel after 3 s, so a hang is reported instead of wedging.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvJitLink.h>
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

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                           \
    }                                                                         \
  } while (0)

typedef int (*probe_fn)(int);

struct Mailbox {
  volatile unsigned long long cmd;    // host writes: seq<<8 | op
  volatile unsigned long long arg;    // function pointer or value
  volatile unsigned long long resp;   // device writes: seq
  volatile long long result;
  volatile unsigned long long t_dev;  // globaltimer at response
};

__device__ __noinline__ int local_triple(int x) { return 3 * x; }
__device__ probe_fn g_local = local_triple;

__device__ __forceinline__ unsigned long long ld_sys(const volatile unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_sys(volatile unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One CTA (thread 0) serves the mailbox; the others idle on a device flag so
// the grid is resident on every SM like the real worker kernel.
__global__ void persistent(Mailbox* mb, volatile int* dev_stop) {
  if (blockIdx.x != 0) {
    while (*dev_stop == 0) __nanosleep(1000);
    return;
  }
  if (threadIdx.x != 0) return;
  unsigned long long last = 0;
  for (;;) {
    unsigned long long c = ld_sys(&mb->cmd);
    if (c == last) continue;
    last = c;
    unsigned op = (unsigned)(c & 0xff);
    long long r = 0;
    if (op == 99) {
      *dev_stop = 1;
      st_sys(&mb->resp, c >> 8);
      return;
    } else if (op == 1) {
      r = 0;
    } else if (op == 2) {
      probe_fn f = (probe_fn)(mb->arg);
      r = f(7);
    } else if (op == 3) {
      r = g_local(7);
    }
    mb->result = r;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    mb->t_dev = t;
    __threadfence_system();
    st_sys(&mb->resp, c >> 8);
  }
}

static Mailbox* g_mb;
static int* g_stop_dev;
static unsigned long long g_seq = 0;
static cudaStream_t g_ks, g_side;

static long long call(unsigned op, unsigned long long arg = 0) {
  g_mb->arg = arg;
  unsigned long long s = ++g_seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  g_mb->cmd = (s << 8) | op;
  auto t0 = std::chrono::steady_clock::now();
  while (g_mb->resp != s) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(5)) {
      std::printf("mailbox timeout op=%u\n", op);
      return -1;
    }
  }
  return g_mb->result;
}

static void launch_persistent(int nsm) {
  CK(cudaMemsetAsync(g_stop_dev, 0, sizeof(int), g_side));
  CK(cudaStreamSynchronize(g_side));
  persistent<<<nsm, 256, 0, g_ks>>>((Mailbox*)g_mb, g_stop_dev);
  CK(cudaGetLastError());
  // wait until it answers
  if (call(1) != 0) std::printf("persistent kernel did not answer\n");
}

static void stop_persistent() {
  unsigned long long s = ++g_seq;
  g_mb->cmd = (s << 8) | 99;
}

// Runs fn; if it has not returned within 3 s, release the persistent kernel
// (which unblocks any implicit device synchronisation) and report a hang.
static bool guarded(const char* name, const std::function<void()>& fn) {
  std::atomic<bool> done{false};
  std::thread wd([&] {
    for (int i = 0; i < 300 && !done.load(); ++i) std::this_thread::sleep_for(std::chrono::milliseconds(10));
    if (!done.load()) stop_persistent();
  });
  auto t0 = std::chrono::steady_clock::now();
  fn();
  double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  done = true;
  wd.join();
  bool alive = cudaStreamQuery(g_ks) == cudaErrorNotReady;
  std::printf("%-34s %9.3f ms  %s\n", name, ms, alive ? "OK (kernel still resident)" : "BLOCKED until kernel exit");
  return alive;
}

static const char* kJitSrc = R"(
extern "C" __device__ __noinline__ int jit_op(int x) { return x * 5 + 1; }
typedef int (*probe_fn)(int);
extern "C" __device__ probe_fn jit_op_ptr = jit_op;
)";

static std::vector<char> jit_cubin(int maxreg, double* ms_rtc, double* ms_link) {
  auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  nvrtcCreateProgram(&prog, kJitSrc, "jit.cu", 0, nullptr, nullptr);
  std::string mr = "--maxrregcount=" + std::to_string(maxreg);
  const char* opts[] = {"-arch=sm_100a", "-rdc=true", "--fmad=false", mr.c_str()};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, 0);
    nvrtcGetProgramLog(prog, log.data());
    std::printf("nvrtc failed: %s\n", log.c_str());
    std::exit(1);
  }
  size_t ltoSize = 0;
  nvrtcGetCUBINSize(prog, &ltoSize);
  std::vector<char> relo(ltoSize);
  nvrtcGetCUBIN(prog, relo.data());
  nvrtcDestroyProgram(&prog);
  auto t1 = std::chrono::steady_clock::now();
  nvJitLinkHandle h;
  const char* lopts[] = {"-arch=sm_100a"};
  if (nvJitLinkCreate(&h, 1, lopts) != NVJITLINK_SUCCESS) std::exit(2);
  if (nvJitLinkAddData(h, NVJITLINK_INPUT_CUBIN, relo.data(), relo.size(), "jit") != NVJITLINK_SUCCESS) std::exit(3);
  if (nvJitLinkComplete(h) != NVJITLINK_SUCCESS) {
    size_t n;
    nvJitLinkGetErrorLogSize(h, &n);
    std::string log(n, 0);
    nvJitLinkGetErrorLog(h, log.data());
    std::printf("link failed: %s\n", log.c_str());
    std::exit(4);
  }
  size_t cs;
  nvJitLinkGetLinkedCubinSize(h, &cs);
  std::vector<char> cubin(cs);
  nvJitLinkGetLinkedCubin(h, cubin.data());
  nvJitLinkDestroy(&h);
  auto t2 = std::chrono::steady_clock::now();
  *ms_rtc = std::chrono::duration<double, std::milli>(t1 - t0).count();
  *ms_link = std::chrono::duration<double, std::milli>(t2 - t1).count();
  return cubin;
}

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  std::printf("device %s sms=%d l2=%d MB concurrentManaged=%d pageable=%d canMapHost=%d\n", prop.name,
              prop.multiProcessorCount, prop.l2CacheSize >> 20, prop.concurrentManagedAccess,
              prop.pageableMemoryAccess, prop.canMapHostMemory);
  CK(cudaDeviceSetLimit(cudaLimitStackSize, 4096));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, persistent));
  std::printf("persistent kernel regs=%d local=%zu\n", fa.numRegs, fa.localSizeBytes);
  CK(cudaStreamCreateWithFlags(&g_ks, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&g_side, cudaStreamNonBlocking));
  CK(cudaHostAlloc(&g_mb, sizeof(Mailbox), cudaHostAllocMapped));
  std::memset((void*)g_mb, 0, sizeof(Mailbox));
  CK(cudaMalloc(&g_stop_dev, sizeof(int)));
  cuInit(0);

  const int nsm = prop.multiProcessorCount;
  launch_persistent(nsm);

  // 1. ping-pong latency
  {
    std::vector<double> lat;
    for (int i = 0; i < 20000; ++i) {
      auto t0 = std::chrono::steady_clock::now();
      call(1);
      lat.push_back(std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
    std::sort(lat.begin(), lat.end());
    std::printf("mailbox round trip: p50 %.3f us p99 %.3f us min %.3f us\n", lat[lat.size() / 2],
                lat[lat.size() * 99 / 100], lat[0]);
  }
  std::printf("local fnptr call -> %lld (expect 21)\n", call(3));

  // 2. API behaviour with the kernel resident
  void* p = nullptr;
  if (!guarded("cudaMalloc 1MB", [&] { CK(cudaMalloc(&p, 1 << 20)); })) launch_persistent(nsm);
  void* pa = nullptr;
  if (!guarded("cudaMallocAsync 1MB (side)", [&] {
        CK(cudaMallocAsync(&pa, 1 << 20, g_side));
        CK(cudaStreamSynchronize(g_side));
      }))
    launch_persistent(nsm);
  if (!guarded("cudaFreeAsync (side)", [&] {
        CK(cudaFreeAsync(pa, g_side));
        CK(cudaStreamSynchronize(g_side));
      }))
    launch_persistent(nsm);
  void* pm = nullptr;
  if (!guarded("cudaMallocManaged 64MB", [&] { CK(cudaMallocManaged(&pm, 64 << 20)); })) launch_persistent(nsm);
  if (!guarded("host touch managed", [&] { std::memset(pm, 1, 64 << 20); })) launch_persistent(nsm);
  if (!guarded("cudaMemPrefetchAsync managed", [&] {
        cudaMemLocation loc{};
        loc.type = cudaMemLocationTypeDevice;
        loc.id = 0;
        CK(cudaMemPrefetchAsync(pm, 64 << 20, loc, 0, g_side));
        CK(cudaStreamSynchronize(g_side));
      }))
    launch_persistent(nsm);
  if (!guarded("cudaMemsetAsync (side)", [&] {
        CK(cudaMemsetAsync(p, 0, 1 << 20, g_side));
        CK(cudaStreamSynchronize(g_side));
      }))
    launch_persistent(nsm);
  void* ph = nullptr;
  if (!guarded("cudaHostAlloc 16MB", [&] { CK(cudaHostAlloc(&ph, 16 << 20, cudaHostAllocMapped)); }))
    launch_persistent(nsm);
  if (!guarded("cudaMemcpyAsync H2D (side)", [&] {
        CK(cudaMemcpyAsync(p, ph, 1 << 20, cudaMemcpyHostToDevice, g_side));
        CK(cudaStreamSynchronize(g_side));
      }))
    launch_persistent(nsm);
  if (!guarded("cudaMemcpy (legacy stream)", [&] { CK(cudaMemcpy(ph, p, 1 << 20, cudaMemcpyDeviceToHost)); }))
    launch_persistent(nsm);

  // 3. JIT module into the live context, call through its pointer.
  double ms_rtc = 0, ms_link = 0;
  std::vector<char> cubin = jit_cubin(fa.numRegs, &ms_rtc, &ms_link);
  std::printf("nvrtc %.2f ms, nvJitLink %.2f ms, cubin %zu B\n", ms_rtc, ms_link, cubin.size());
  CUmodule mod = nullptr;
  if (!guarded("cuModuleLoadData", [&] {
        CUresult r = cuModuleLoadData(&mod, cubin.data());
        if (r != CUDA_SUCCESS) std::printf("cuModuleLoadData err %d\n", (int)r);
      }))
    launch_persistent(nsm);
  CUdeviceptr gp;
  size_t gsz;
  CUresult rr = cuModuleGetGlobal(&gp, &gsz, mod, "jit_op_ptr");
  std::printf("cuModuleGetGlobal -> %d size %zu\n", (int)rr, gsz);
  unsigned long long fnv = 0;
  guarded("read fn ptr via memcpyAsync", [&] {
    CK(cudaMemcpyAsync(&fnv, (void*)gp, 8, cudaMemcpyDeviceToHost, g_side));
    CK(cudaStreamSynchronize(g_side));
  });
  std::printf("jit fn ptr = 0x%llx\n", fnv);
  long long r = call(2, fnv);
  std::printf("cross-module fnptr call -> %lld (expect 36)\n", r);
  cudaError_t ke = cudaStreamQuery(g_ks);
  std::printf("kernel state after call: %s\n", cudaGetErrorString(ke));

  if (!guarded("cudaFree (device)", [&] { CK(cudaFree(p)); })) launch_persistent(nsm);
  if (!guarded("cudaFree (managed)", [&] { CK(cudaFree(pm)); })) launch_persistent(nsm);

  stop_persistent();
  CK(cudaStreamSynchronize(g_ks));
  std::printf("probe done\n");
  return 0;
}
