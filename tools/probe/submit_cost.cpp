// Producer-side cost breakdown of Runtime::submit on the GPU box.
//   build/probe/submit_cost
// Prints ns/task for: the full submit (workers live), the full submit with
// workers held (no device traffic on the ring), and the pieces: TensorView
// copies, cell acquire, ring reserve+publish of a prebuilt slot.
#include <algorithm>
#include <array>
#include <atomic>
#include <cctype>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <future>
#include <immintrin.h>
#include <initializer_list>
#include <istream>
#include <map>
#include <memory>
#include <mutex>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>
#define private public  // probe only: time the submit path's internal steps
#include <gpuos/runtime.hpp>
#undef private

#include <chrono>
#include <cstdio>
#include <vector>

using namespace gpuos;

static double now_ns() {
  return std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  RuntimeConfig cfg;
  cfg.capacity = 16384;
  cfg.telemetry_enabled = false;
  Runtime rt(cfg);
  const int n = 10000, e = 4096;
  TensorView A = rt.alloc_tensor(DType::F32, {int64_t(n) * e});
  TensorView B = rt.alloc_tensor(DType::F32, {int64_t(n) * e});
  TensorView Cv = rt.alloc_tensor(DType::F32, {int64_t(n) * e});
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
  gpuos_dev* dev = rt.device();
  for (int rep = 0; rep < 4; ++rep) {
    // 1. live workers
    double t0 = now_ns();
    for (int i = 0; i < n; ++i) rt.submit(OpKind::Add, {a[i], b[i]}, c[i]);
    double t1 = now_ns();
    rt.wait_all();
    double t2 = now_ns();
    std::printf("live: submit %.1f ns/task, drain %.1f us\n", (t1 - t0) / n, (t2 - t1) / 1e3);
    // 2. held workers (ring fills, no device reads racing the producer)
    gpuos_dev_hold(dev, 1);
    t0 = now_ns();
    for (int i = 0; i < n; ++i) rt.submit(OpKind::Add, {a[i], b[i]}, c[i]);
    t1 = now_ns();
    gpuos_dev_hold(dev, 0);
    rt.wait_all();
    std::printf("held: submit %.1f ns/task\n", (t1 - t0) / n);
    // 2b. handles kept (no destructor in the loop)
    {
      std::vector<TaskHandle> keep;
      keep.reserve(n);
      t0 = now_ns();
      for (int i = 0; i < n; ++i) keep.push_back(rt.submit(OpKind::Add, {a[i], b[i]}, c[i]));
      t1 = now_ns();
      rt.wait_all();
      const double t2k = now_ns();
      keep.clear();
      const double t3k = now_ns();
      std::printf("kept handles: submit %.1f ns/task, dtor %.1f ns/task\n", (t1 - t0) / n, (t3k - t2k) / n);
    }
    // 2c. internal steps of submit_span, each in its own loop
    {
      std::vector<uint32_t> cells(n);
      t0 = now_ns();
      for (int i = 0; i < n; ++i) cells[i] = rt.cells_->acquire(rt.next_id_++);
      t1 = now_ns();
      double t_acq = (t1 - t0) / n;
      for (int i = 0; i < n; ++i) rt.cells_->release(cells[i]);  // the handle-less acquires' references
      volatile int sinkv = 0;
      t0 = now_ns();
      for (int i = 0; i < n; ++i) {
        const TensorView in2[2] = {a[i], b[i]};
        sinkv += (int)rt.validate(std::span<const TensorView>(in2, 2), c[i], std::span<const double>());
        sinkv += rt.eligible(0, std::span<const TensorView>(in2, 2), c[i]);
      }
      t1 = now_ns();
      double t_val = (t1 - t0) / n;
      alignas(64) gpuos_task tk;
      t0 = now_ns();
      for (int i = 0; i < n; ++i) {
        const TensorView in2[2] = {a[i], b[i]};
        rt.build_task(0, std::span<const TensorView>(in2, 2), c[i], std::span<const double>(), cells[i], 5, 0, &tk);
      }
      t1 = now_ns();
      double t_build = (t1 - t0) / n;
      std::printf("steps: cell acquire %.1f, validate+eligible %.1f, build_task %.1f ns/task\n", t_acq, t_val, t_build);
      for (int i = 0; i < n; ++i) rt.cells_->complete(cells[i], 0, ErrorCode::Ok);
    }
    // 3. TensorView copies only
    t0 = now_ns();
    volatile size_t sink = 0;
    for (int i = 0; i < n; ++i) {
      std::initializer_list<TensorView> il = {a[i], b[i]};
      sink += il.begin()->shape.size();
    }
    t1 = now_ns();
    std::printf("views: %.1f ns/task\n", (t1 - t0) / n);
    // 4. raw reserve + publish of one prebuilt slot
    alignas(64) gpuos_task t;
    std::memset(&t, 0, sizeof(t));
    t.op_id = 2;  // relu of nothing: n_inputs 0 -> ArityError, cheap on device
    gpuos_dev_hold(dev, 1);
    t0 = now_ns();
    int pub = 0;
    for (int i = 0; i < n; ++i) {
      uint64_t pos;
      if (gpuos_ring_reserve(dev, &pos) != 0) break;
      t.seq = 1000000 + i;
      gpuos_ring_publish(dev, pos, &t);
      ++pub;
    }
    t1 = now_ns();
    gpuos_dev_hold(dev, 0);
    std::printf("raw publish (held): %.1f ns/task (%d)\n", (t1 - t0) / pub, pub);
    // wait for those raw tasks: processed count covers them
    gpuos_snapshot s{};
    for (;;) {
      gpuos_ring_peek(dev, &s);
      if (s.processed >= s.tail) break;
    }
    t0 = now_ns();
    for (int i = 0; i < n; ++i) {
      uint64_t pos;
      while (gpuos_ring_reserve(dev, &pos) != 0) {}
      t.seq = 2000000 + i;
      gpuos_ring_publish(dev, pos, &t);
    }
    t1 = now_ns();
    for (;;) {
      gpuos_ring_peek(dev, &s);
      if (s.processed >= s.tail) break;
    }
    std::printf("raw publish (live): %.1f ns/task\n", (t1 - t0) / n);
  }
  return 0;
}
