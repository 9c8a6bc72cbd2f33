// Benchmark driver for bench.py (built as libgpuos_bench.so, called via ctypes
// so bench.py keeps the multi-rank barriers and JSON contract).
//
// Workload "config1" (BASELINE.json configs[0]/[1] headline): N fp32 Add
// tasks of E contiguous elements, distinct a_i, b_i, c_i per task carved from
// three large buffers (3 * N * E * 4 bytes, 491.5 MB at 10,000 x 4096, far
// above the 126 MB L2), submitted through gpuos::Runtime::submit.
//
// Modes of one step:
//   0  persistent  : worker kernel launched at step start, N submits, wait_all,
//                    sentinel; device time = CUDA events bracketing the worker
//                    kernel's lifetime on its own stream.
//   1  per-op      : baseline (a), one cudaLaunchKernel of the same task body
//                    per task, back to back on one stream; CUDA-event timed.
//   3  lean per-op : a minimal dense f32 add kernel per task (gpuos_launch_lean_add)
//   2  e2e         : like 0 but inputs start in pinned host memory and outputs
//                    end there: chunked H2D copies, submits and per-chunk D2H
//                    copies, pipelined, all inside the (host-clock) timed region.
#include <gpuos/runtime.hpp>
#include <immintrin.h>

#include "oracle_check.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

using namespace gpuos;

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Bench {
  std::unique_ptr<Runtime> rt;
  gpuos_dev* dev = nullptr;
  int n = 0, e = 0;
  TensorView A, B, Cv;                 // whole buffers
  std::vector<TensorView> a, b, c;     // per-task views
  float* hA = nullptr;                 // pinned host copies (e2e)
  float* hB = nullptr;
  float* hC = nullptr;
  void* kstream = nullptr;
  void* lstream = nullptr;   // per-op launch stream
  void* cstream = nullptr;   // copy stream (H2D)
  void* dstream = nullptr;   // copy stream (D2H)
  void* ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<float> expect;  // expected c = a + b: the oracle's add once loaded (f32(a + b) before)
  bool expect_from_oracle = false;
  uint64_t last_fallbacks = 0;
};

uint64_t config_seed(uint64_t seed, uint64_t config) {  // bench.hpp:280-282
  return seed ^ (config * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull);
}

}  // namespace

extern "C" {

void* gb_open(int device, int n_tasks, int n_elems, int workers, int capacity) {
  auto* b = new Bench();
  RuntimeConfig cfg;
  cfg.device = device;
  cfg.capacity = capacity > 0 ? static_cast<size_t>(capacity) : 4096;
  cfg.workers.num_workers = workers > 0 ? static_cast<size_t>(workers) : 0;
  // the trace ring is off on the measured path; GPUOS_BENCH_TRACE=1 turns it
  // on to print per-phase device stamps after each step (diagnostics only)
  cfg.telemetry_enabled = std::getenv("GPUOS_BENCH_TRACE") != nullptr;
  // plain device memory for the task buffers: the e2e arm moves 491.5 MB per
  // step over PCIe, and copies into managed memory measured ~25% slower
  cfg.device_buffers = true;
  b->rt = std::make_unique<Runtime>(cfg);
  b->dev = b->rt->device();
  b->n = n_tasks;
  b->e = n_elems;
  const int64_t total = static_cast<int64_t>(n_tasks) * n_elems;
  b->A = b->rt->alloc_tensor(DType::F32, {total});
  b->B = b->rt->alloc_tensor(DType::F32, {total});
  b->Cv = b->rt->alloc_tensor(DType::F32, {total});
  for (int i = 0; i < n_tasks; ++i) {
    TensorView va = b->A, vb = b->B, vc = b->Cv;
    va.shape = vb.shape = vc.shape = {static_cast<int64_t>(n_elems)};
    va.strides = vb.strides = vc.strides = {1};
    va.offset = vb.offset = vc.offset = static_cast<int64_t>(i) * n_elems;
    b->a.push_back(va);
    b->b.push_back(vb);
    b->c.push_back(vc);
  }
  check_abi(gpuos_host_alloc(b->dev, total * 4, reinterpret_cast<void**>(&b->hA)), "host alloc");
  check_abi(gpuos_host_alloc(b->dev, total * 4, reinterpret_cast<void**>(&b->hB)), "host alloc");
  check_abi(gpuos_host_alloc(b->dev, total * 4, reinterpret_cast<void**>(&b->hC)), "host alloc");
  // seeded U(-1,1) narrowed to f32 (bench.hpp:210-215, seed 42, config 1)
  std::mt19937_64 rng(config_seed(42, 1));
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  b->expect.resize(static_cast<size_t>(total));
  for (int64_t i = 0; i < total; ++i) b->hA[i] = static_cast<float>(dist(rng));
  for (int64_t i = 0; i < total; ++i) b->hB[i] = static_cast<float>(dist(rng));
  for (int64_t i = 0; i < total; ++i) b->expect[static_cast<size_t>(i)] = b->hA[i] + b->hB[i];
  b->rt->pool().upload(b->A.buffer, b->hA, total * 4);
  b->rt->pool().upload(b->B.buffer, b->hB, total * 4);
  b->rt->pool().prefetch(b->A.buffer);
  b->rt->pool().prefetch(b->B.buffer);
  b->rt->pool().prefetch(b->Cv.buffer);
  check_abi(gpuos_dev_kernel_stream(b->dev, &b->kstream), "kernel stream");
  check_abi(gpuos_stream_create(b->dev, &b->lstream), "launch stream");
  check_abi(gpuos_stream_create(b->dev, &b->cstream), "copy stream");
  check_abi(gpuos_stream_create(b->dev, &b->dstream), "d2h stream");
  for (void*& e : b->ev) check_abi(gpuos_event_create(b->dev, &e), "event");
  // steps start the worker kernel themselves
  b->rt->wait_all();
  check_abi(gpuos_dev_stop(b->dev), "stop");
  return b;
}

// out: [0] device ms (events), [1] host ms, [2] tasks, [3] algorithmic bytes,
//      [4] queue-full fallbacks during the step, [5] host ms spent in submit() calls
int gb_step(void* h, int mode, double* out) {
  auto* b = static_cast<Bench*>(h);
  out[5] = 0;
  Runtime& rt = *b->rt;
  const uint64_t fb0 = rt.counters().queue_full_fallbacks;
  double dev_ms = 0, host_ms = 0;
  if (mode == 0 || mode == 2) {
    check_abi(gpuos_event_record(b->dev, b->ev[0], b->kstream), "ev0");
    check_abi(gpuos_dev_start(b->dev), "start");
    check_abi(gpuos_event_record(b->dev, b->ev[1], b->kstream), "ev1");  // completes at kernel exit
    const double t0 = now_ms();
    if (mode == 0) {
      for (int i = 0; i < b->n; ++i) rt.submit(OpKind::Add, {b->a[i], b->b[i]}, b->c[i]);
      out[5] = now_ms() - t0;  // producer-side cost of the N submits
      // the shutdown sentinel goes right behind the batch: the generation
      // drains every committed task, then exits (ev1), so the device-timed
      // step ends when the last task completes, not when the host's
      // wait_all poll notices it
      check_abi(gpuos_dev_stop(b->dev), "stop");
      rt.wait_all();
    } else {
      // e2e: a three-stage pipeline over chunks of tasks -- H2D of chunk k+1
      // (copy stream) overlaps the tasks of chunk k, and the D2H of every
      // finished chunk (second copy stream) overlaps both, so the step is
      // bounded by the H2D volume over PCIe rather than H2D + D2H in series.
      const char* ce = std::getenv("GB_E2E_CHUNKS");
      const int chunks = ce ? std::max(1, std::atoi(ce)) : 16;
      const int per = (b->n + chunks - 1) / chunks;
      const BufferPool::Buffer& ba = rt.pool().lookup(b->A.buffer);
      const BufferPool::Buffer& bb = rt.pool().lookup(b->B.buffer);
      const BufferPool::Buffer& bc = rt.pool().lookup(b->Cv.buffer);
      std::vector<void*> evs(chunks, nullptr);
      auto span_of = [&](int k, uint64_t* off, uint64_t* bytes) {
        const int lo = k * per, hi = std::min(b->n, lo + per);
        *off = static_cast<uint64_t>(lo) * b->e * 4;
        *bytes = hi > lo ? static_cast<uint64_t>(hi - lo) * b->e * 4 : 0;
        return hi > lo;
      };
      for (int k = 0; k < chunks; ++k) {
        uint64_t off, bytes;
        if (!span_of(k, &off, &bytes)) break;
        check_abi(gpuos_copy_async(b->dev, static_cast<char*>(ba.data) + off, reinterpret_cast<char*>(b->hA) + off, bytes, 0, b->cstream), "h2d");
        check_abi(gpuos_copy_async(b->dev, static_cast<char*>(bb.data) + off, reinterpret_cast<char*>(b->hB) + off, bytes, 0, b->cstream), "h2d");
        check_abi(gpuos_event_create(b->dev, &evs[k]), "ev");
        check_abi(gpuos_event_record(b->dev, evs[k], b->cstream), "ev");
      }
      std::vector<TaskHandle> hs;
      hs.reserve(static_cast<size_t>(b->n));
      // one host loop, never blocking: submit a chunk as soon as its inputs
      // landed, start a chunk's D2H as soon as its last task completed
      int next_sub = 0, next_out = 0, scan = 0;
      int nchunks = 0;
      for (int k = 0; k < chunks; ++k) nchunks += (k * per < b->n) ? 1 : 0;
      while (next_out < nchunks) {
        if (next_sub < nchunks && gpuos_event_done(b->dev, evs[next_sub])) {
          const int lo = next_sub * per, hi = std::min(b->n, lo + per);
          for (int i = lo; i < hi; ++i) hs.push_back(rt.submit(OpKind::Add, {b->a[i], b->b[i]}, b->c[i]));
          ++next_sub;
          continue;
        }
        if (next_out < next_sub) {
          const int hi = std::min(b->n, (next_out + 1) * per);
          while (scan < hi && hs[static_cast<size_t>(scan)].state() != TaskState::Pending) ++scan;
          if (scan == hi) {
            uint64_t off, bytes;
            if (span_of(next_out, &off, &bytes))
              check_abi(gpuos_copy_async(b->dev, reinterpret_cast<char*>(b->hC) + off, static_cast<char*>(bc.data) + off, bytes, 1, b->dstream), "d2h");
            ++next_out;
            continue;
          }
        }
        _mm_pause();
      }
      check_abi(gpuos_stream_sync(b->dev, b->dstream), "sync");
      for (void* e : evs)
        if (e) gpuos_event_destroy(b->dev, e);
    }
    const double t1 = now_ms();
    if (mode != 0) check_abi(gpuos_dev_stop(b->dev), "stop");
    if (std::getenv("GPUOS_BENCH_TRACE")) {
      std::vector<gpuos_trace_phase> ph(static_cast<size_t>(b->n));
      uint64_t n = 0;
      gpuos_trace_phases(b->dev, ph.data(), ph.size(), &n);
      auto pct = [&](auto f, double q) {
        std::vector<double> v;
        for (uint64_t i = 0; i < n; ++i) v.push_back(f(ph[i]));
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[static_cast<size_t>(q * (v.size() - 1))];
      };
      auto enq_seen = [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.seen_ns - p.enqueue_ns) / 1e3; };
      auto seen_deq = [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.dequeue_ns - p.seen_ns) / 1e3; };
      auto exec = [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.end_ns - p.dequeue_ns) / 1e3; };
      auto done = [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.done_ns - p.end_ns) / 1e3; };
      auto tick = [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.seen_ns - p.ticket_ns) / 1e3; };
      uint64_t first = UINT64_MAX, last = 0;
      for (uint64_t i = 0; i < n; ++i) {
        first = std::min(first, ph[i].seen_ns);
        last = std::max(last, ph[i].done_ns);
      }
      std::fprintf(stderr,
                   "trace n=%llu span %.3f ms | enq->seen p50 %.2f p90 %.2f | seen->deq p50 %.2f p90 %.2f | exec p50 "
                   "%.2f p90 %.2f | done p50 %.2f | ticket->seen p50 %.2f us\n",
                   (unsigned long long)n, (last - first) / 1e6, pct(enq_seen, .5), pct(enq_seen, .9), pct(seen_deq, .5),
                   pct(seen_deq, .9), pct(exec, .5), pct(exec, .9), pct(done, .5), pct(tick, .5));
      // step timeline: tasks enqueued / seen / done per 25 us bucket, from
      // the first ticket (the generation's first claim)
      uint64_t t_first = UINT64_MAX;
      for (uint64_t i = 0; i < n; ++i) t_first = std::min({t_first, ph[i].ticket_ns, ph[i].enqueue_ns});
      const int nb = 48;
      std::vector<int> enq(nb), seen(nb), dn(nb);
      auto bk = [&](uint64_t t) { return std::min<int>(nb - 1, (int)((t - t_first) / 25000)); };
      for (uint64_t i = 0; i < n; ++i) {
        ++enq[bk(ph[i].enqueue_ns)];
        ++seen[bk(ph[i].seen_ns)];
        ++dn[bk(ph[i].done_ns)];
      }
      std::fprintf(stderr, "timeline (25 us buckets from the first claim/enqueue): enq/seen/done\n");
      for (int k = 0; k < nb; ++k)
        if (enq[k] || seen[k] || dn[k]) std::fprintf(stderr, "  %4d us: %5d %5d %5d\n", 25 * k, enq[k], seen[k], dn[k]);
    }
    float ms = 0;
    check_abi(gpuos_event_sync(b->dev, b->ev[1]), "sync ev1");
    check_abi(gpuos_event_elapsed_ms(b->dev, b->ev[0], b->ev[1], &ms), "elapsed");
    dev_ms = ms;
    host_ms = t1 - t0;
  } else if (mode == 3) {
    // lean per-op baseline: a minimal add kernel per task (4 parameters, no
    // descriptor, no dynamic shared memory, no table lookup, no lock)
    const BufferPool::Buffer& ba = rt.pool().lookup(b->A.buffer);
    const BufferPool::Buffer& bb = rt.pool().lookup(b->B.buffer);
    const BufferPool::Buffer& bc = rt.pool().lookup(b->Cv.buffer);
    check_abi(gpuos_event_record(b->dev, b->ev[2], b->lstream), "ev2");
    const double t0 = now_ms();
    for (int i = 0; i < b->n; ++i) {
      const uint64_t off = static_cast<uint64_t>(i) * b->e * 4;
      check_abi(gpuos_launch_lean_add(b->dev, static_cast<char*>(bc.data) + off, static_cast<char*>(ba.data) + off,
                                      static_cast<char*>(bb.data) + off, b->e, b->lstream),
                "lean launch");
    }
    check_abi(gpuos_event_record(b->dev, b->ev[3], b->lstream), "ev3");
    check_abi(gpuos_stream_sync(b->dev, b->lstream), "sync");
    const double t1 = now_ms();
    float ms = 0;
    check_abi(gpuos_event_elapsed_ms(b->dev, b->ev[2], b->ev[3], &ms), "elapsed");
    dev_ms = ms;
    host_ms = t1 - t0;
  } else {
    // baseline (a): the same bodies, one launch per task
    alignas(64) gpuos_task t;
    std::memset(&t, 0, sizeof(t));
    t.op_id = static_cast<uint32_t>(OpKind::Add);
    t.n_inputs = 2;
    t.size = static_cast<uint64_t>(b->e);
    const BufferPool::Buffer& ba = rt.pool().lookup(b->A.buffer);
    const BufferPool::Buffer& bb = rt.pool().lookup(b->B.buffer);
    const BufferPool::Buffer& bc = rt.pool().lookup(b->Cv.buffer);
    for (int v = 0; v < 3; ++v) {
      t.views[v].rank = 1;
      t.views[v].extents[0] = b->e;
      t.views[v].strides[0] = 1;
      t.views[v].dtype = GPUOS_F32;
    }
    check_abi(gpuos_event_record(b->dev, b->ev[2], b->lstream), "ev2");
    const double t0 = now_ms();
    for (int i = 0; i < b->n; ++i) {
      const uint64_t off = static_cast<uint64_t>(i) * b->e * 4;
      t.seq = static_cast<uint64_t>(i) + 1;
      t.views[0].addr = reinterpret_cast<uint64_t>(static_cast<char*>(bc.data) + off);
      t.views[1].addr = reinterpret_cast<uint64_t>(static_cast<char*>(ba.data) + off);
      t.views[2].addr = reinterpret_cast<uint64_t>(static_cast<char*>(bb.data) + off);
      check_abi(gpuos_launch_task(b->dev, &t, b->lstream), "launch");
    }
    check_abi(gpuos_event_record(b->dev, b->ev[3], b->lstream), "ev3");
    check_abi(gpuos_stream_sync(b->dev, b->lstream), "sync");
    const double t1 = now_ms();
    float ms = 0;
    check_abi(gpuos_event_elapsed_ms(b->dev, b->ev[2], b->ev[3], &ms), "elapsed");
    dev_ms = ms;
    host_ms = t1 - t0;
  }
  out[0] = dev_ms;
  out[1] = host_ms;
  out[2] = b->n;
  out[3] = static_cast<double>(b->n) * b->e * 12.0;  // 2 reads + 1 write of 4 bytes per element
  out[4] = static_cast<double>(rt.counters().queue_full_fallbacks - fb0);
  return 0;
}

// Queue-depth-1 latency: submit -> wait (mode 0) or launch -> sync (mode 1).
// out: [0] p50 us, [1] p99 us, [2] mean us
int gb_latency(void* h, int mode, int samples, int warmup, double* out) {
  auto* b = static_cast<Bench*>(h);
  Runtime& rt = *b->rt;
  std::vector<double> lat;
  lat.reserve(static_cast<size_t>(samples));
  if (mode == 0) check_abi(gpuos_dev_start(b->dev), "start");
  alignas(64) gpuos_task t;
  std::memset(&t, 0, sizeof(t));
  const BufferPool::Buffer& ba = rt.pool().lookup(b->A.buffer);
  const BufferPool::Buffer& bb = rt.pool().lookup(b->B.buffer);
  const BufferPool::Buffer& bc = rt.pool().lookup(b->Cv.buffer);
  t.op_id = static_cast<uint32_t>(OpKind::Add);
  t.n_inputs = 2;
  t.size = static_cast<uint64_t>(b->e);
  for (int v = 0; v < 3; ++v) {
    t.views[v].rank = 1;
    t.views[v].extents[0] = b->e;
    t.views[v].strides[0] = 1;
    t.views[v].dtype = GPUOS_F32;
  }
  for (int s = 0; s < samples + warmup; ++s) {
    const int i = s % b->n;
    const double t0 = now_ms();
    if (mode == 0) {
      TaskHandle th = rt.submit(OpKind::Add, {b->a[i], b->b[i]}, b->c[i]);
      const double w0 = now_ms();
      while (th.state() == TaskState::Pending) {
        if (now_ms() - w0 > 5000) {
          char dbg[2048];
          gpuos_dev_debug(b->dev, dbg, sizeof(dbg));
          std::fprintf(stderr, "gb_latency: task %llu stalled: %s\n", (unsigned long long)th.id(), dbg);
          return 1;
        }
      }
    } else {
      const uint64_t off = static_cast<uint64_t>(i) * b->e * 4;
      t.views[0].addr = reinterpret_cast<uint64_t>(static_cast<char*>(bc.data) + off);
      t.views[1].addr = reinterpret_cast<uint64_t>(static_cast<char*>(ba.data) + off);
      t.views[2].addr = reinterpret_cast<uint64_t>(static_cast<char*>(bb.data) + off);
      check_abi(gpuos_launch_task(b->dev, &t, b->lstream), "launch");
      check_abi(gpuos_stream_sync(b->dev, b->lstream), "sync");
    }
    const double t1 = now_ms();
    if (s >= warmup) lat.push_back((t1 - t0) * 1e3);
  }
  if (mode == 0) {
    rt.wait_all();
    check_abi(gpuos_dev_stop(b->dev), "stop");
  }
  std::sort(lat.begin(), lat.end());
  double sum = 0;
  for (double x : lat) sum += x;
  out[0] = lat[lat.size() / 2];
  out[1] = lat[std::min(lat.size() - 1, lat.size() * 99 / 100)];
  out[2] = sum / static_cast<double>(lat.size());
  return 0;
}

// Poison the outputs before a verified step (0xff bytes = NaN): the device
// copy, and for the e2e arm also the pinned host copy the D2H lands in.
int gb_poison(void* h) {
  auto* b = static_cast<Bench*>(h);
  b->rt->pool().fill(b->Cv.buffer, 0xff);
  std::memset(b->hC, 0xff, static_cast<size_t>(b->n) * b->e * 4);
  return 0;
}

// Bit-exact self-check of every output element against f32(a + b).
int gb_verify(void* h, uint64_t* mismatches, uint64_t* checked, int from_host_copy) {
  auto* b = static_cast<Bench*>(h);
  const uint64_t total = static_cast<uint64_t>(b->n) * b->e;
  if (gbcheck::oracle().ok && !b->expect_from_oracle) {  // the checker's add over the same inputs
    const int64_t t = static_cast<int64_t>(total);
    orc_view o = gbcheck::view(b->expect.data(), ORC_F32, 0, {t}, {1});
    orc_view in[2] = {gbcheck::view(b->hA, ORC_F32, 0, {t}, {1}), gbcheck::view(b->hB, ORC_F32, 0, {t}, {1})};
    if (gbcheck::oracle().elementwise(0, &o, in, 2) != 0) return 1;
    b->expect_from_oracle = true;
  }
  std::vector<float> got(total);
  if (from_host_copy) std::memcpy(got.data(), b->hC, total * 4);
  else b->rt->pool().download(b->Cv.buffer, got.data(), total * 4);
  uint64_t bad = 0;
  for (uint64_t i = 0; i < total; ++i)
    if (std::memcmp(&got[i], &b->expect[i], 4) != 0) ++bad;
  *mismatches = bad;
  *checked = total;
  return 0;
}

int gb_checker(void* h) { return static_cast<Bench*>(h)->expect_from_oracle ? 1 : 0; }

int gb_info(void* h, char* buf, size_t cap) {
  auto* b = static_cast<Bench*>(h);
  uint32_t sms = 0, workers = 0;
  gpuos_dev_sm_count(b->dev, &sms);
  gpuos_dev_num_workers(b->dev, &workers);
  uint64_t capq = 0;
  gpuos_ring_capacity(b->dev, &capq);
  std::snprintf(buf, cap, "{\"sms\": %u, \"workers\": %u, \"threads_per_worker\": 256, \"ring_capacity\": %llu}", sms,
                workers, static_cast<unsigned long long>(capq));
  return 0;
}

void gb_close(void* h) {
  delete static_cast<Bench*>(h);  // workers are already stopped; Runtime shutdown is a no-op drain
}

}  // extern "C"
