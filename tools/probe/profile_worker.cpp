// Finite worker generation for ncu and device-capacity measurement.
//   build/probe/profile_worker [tasks=10000] [elems=4096] [reps=1]
// Config-1 tasks (fp32 Add, distinct buffers) are submitted through
// Runtime::submit while the worker kernel is stopped, then one generation
// drains the ring (sentinel last) and exits: the kernel duration is the
// device-side capacity with no host producer in the loop.
#include <gpuos/runtime.hpp>

#include <cstdio>
#include <cstdlib>
#include <vector>

using namespace gpuos;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 10000;
  const int e = argc > 2 ? std::atoi(argv[2]) : 4096;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 1;
  RuntimeConfig cfg;
  cfg.capacity = static_cast<size_t>(n) + 2;
  cfg.telemetry_enabled = false;
  Runtime rt(cfg);
  const int64_t total = int64_t(n) * e;
  TensorView A = rt.alloc_tensor(DType::F32, {total});
  TensorView B = rt.alloc_tensor(DType::F32, {total});
  TensorView Cv = rt.alloc_tensor(DType::F32, {total});
  std::vector<float> ha(total), hb(total);
  for (int64_t i = 0; i < total; ++i) {
    ha[i] = float((i * 7919) % 2001 - 1000) / 1000.f;
    hb[i] = float((i * 104729) % 1999 - 999) / 999.f;
  }
  rt.pool().upload(A.buffer, ha.data(), total * 4);
  rt.pool().upload(B.buffer, hb.data(), total * 4);
  rt.pool().prefetch(A.buffer);
  rt.pool().prefetch(B.buffer);
  rt.pool().prefetch(Cv.buffer);
  std::vector<TensorView> a, b, c;
  for (int i = 0; i < n; ++i) {
    TensorView va = A, vb = B, vc = Cv;
    va.shape = vb.shape = vc.shape = {int64_t(e)};
    va.strides = vb.strides = vc.strides = {1};
    va.offset = vb.offset = vc.offset = int64_t(i) * e;
    a.push_back(va);
    b.push_back(vb);
    c.push_back(vc);
  }
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  for (int r = 0; r < reps; ++r) {
    for (int i = 0; i < n; ++i) rt.submit(OpKind::Add, {a[i], b[i]}, c[i]);
    float ms = 0;
    check_abi(gpuos_dev_run_finite(rt.device(), &ms), "run_finite");
    const double bytes = double(n) * e * 12.0;
    std::printf("{\"tasks\": %d, \"elems\": %d, \"kernel_ms\": %.4f, \"tasks_per_s\": %.1f, \"alg_GBps\": %.1f}\n", n, e,
                ms, n / (ms / 1e3), bytes / (ms / 1e3) / 1e9);
  }
  std::vector<float> got(total);
  rt.pool().download(Cv.buffer, got.data(), total * 4);
  int64_t bad = 0;
  for (int64_t i = 0; i < total; ++i)
    if (got[i] != ha[i] + hb[i]) ++bad;
  std::printf("mismatches %lld of %lld\n", (long long)bad, (long long)total);
  return bad != 0;
}
