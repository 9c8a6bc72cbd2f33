// Finite worker generation for ncu and device-capacity measurement.
//   build/probe/profile_worker [tasks=10000] [elems=4096] [reps=1]
// Config-1 tasks (fp32 Add, distinct buffers) are submitted through
// Runtime::submit while the worker kernel is stopped, then one generation
// drains the ring (sentinel last) and exits: the kernel duration is the
// device-side capacity with no host producer in the loop.
#include <gpuos/runtime.hpp>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

using namespace gpuos;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 10000;
  const int e = argc > 2 ? std::atoi(argv[2]) : 4096;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 1;
  RuntimeConfig cfg;
  cfg.capacity = static_cast<size_t>(n) + 2;
  const bool trace = std::getenv("PROFILE_TRACE") != nullptr;
  cfg.telemetry_enabled = trace;
  cfg.trace_capacity = static_cast<size_t>(n) + 16;
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
  // PW_OP=matmul_bf16: n bf16 matmul tasks (128x64 . 64x128, K as a
  // transposed view) for tensor-pipe evidence instead of config-1 adds
  const char* pw = std::getenv("PW_OP");
  if (pw && (std::string(pw) == "matmul_bf16" || std::string(pw) == "matmul_f32")) {
    const DType mdt = std::string(pw) == "matmul_f32" ? DType::F32 : DType::BF16;
    const int64_t M = 128, K = 64, N = 128;
    const int nb = 256;  // distinct operand sets, reused round robin
    TensorView QA = rt.alloc_tensor(mdt, {int64_t{nb} * M * K});
    TensorView KB = rt.alloc_tensor(mdt, {int64_t{nb} * N * K});
    TensorView OS = rt.alloc_tensor(mdt, {int64_t{n} * M * N});
    for (int r = 0; r < reps; ++r) {
      for (int i = 0; i < n; ++i) {
        TensorView a2 = QA, b2 = KB, o2 = OS;
        a2.shape = {M, K};
        a2.strides = {K, 1};
        a2.offset = int64_t(i % nb) * M * K;
        b2.shape = {K, N};
        b2.strides = {1, K};
        b2.offset = int64_t(i % nb) * N * K;
        o2.shape = {M, N};
        o2.strides = {N, 1};
        o2.offset = int64_t(i) * M * N;
        rt.submit(OpKind::MatMulSmall, {a2, b2}, o2);
      }
      float ms = 0;
      check_abi(gpuos_dev_run_finite(rt.device(), &ms), "run_finite");
      const double flops = 2.0 * M * N * K * n;
      std::printf("{\"tasks\": %d, \"op\": \"%s 128x64x128\", \"kernel_ms\": %.4f, \"tasks_per_s\": %.1f, "
                  "\"TFLOPs\": %.3f}\n", n, pw, ms, n / (ms / 1e3), flops / (ms / 1e3) / 1e12);
    }
    return 0;
  }
  for (int r = 0; r < reps; ++r) {
    for (int i = 0; i < n; ++i) rt.submit(OpKind::Add, {a[i], b[i]}, c[i]);
    float ms = 0;
    check_abi(gpuos_dev_run_finite(rt.device(), &ms), "run_finite");
    const double bytes = double(n) * e * 12.0;
    std::printf("{\"tasks\": %d, \"elems\": %d, \"kernel_ms\": %.4f, \"tasks_per_s\": %.1f, \"alg_GBps\": %.1f}\n", n, e,
                ms, n / (ms / 1e3), bytes / (ms / 1e3) / 1e9);
    if (trace) {
      std::vector<gpuos_trace_phase> ph(static_cast<size_t>(n));
      uint64_t got = 0;
      gpuos_trace_phases(rt.device(), ph.data(), ph.size(), &got);
      auto pct = [&](auto f, double q) {
        std::vector<double> v;
        for (uint64_t i = 0; i < got; ++i) v.push_back(f(ph[i]));
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[static_cast<size_t>(q * (v.size() - 1))];
      };
      auto show = [&](const char* name, auto f) {
        std::printf("  %-20s p10 %7.2f p50 %7.2f p90 %7.2f us\n", name, pct(f, .1), pct(f, .5), pct(f, .9));
      };
      show("fetch(poll..staged)", [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.dequeue_ns - p.ticket_ns) / 1e3; });
      show("  poll..seen", [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.seen_ns - p.ticket_ns) / 1e3; });
      show("queue(staged..wake)", [](const gpuos_trace_phase& p) { return p.reserved / 1e3; });
      show("exec(wake..end)", [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.end_ns - p.dequeue_ns) / 1e3 - p.reserved / 1e3; });
      show("complete(end..done)", [](const gpuos_trace_phase& p) { return (double)(int64_t)(p.done_ns - p.end_ns) / 1e3; });
      // per-worker spacing between consecutive tickets (claim cadence)
      std::vector<double> gaps;
      std::vector<gpuos_trace_phase> v(ph.begin(), ph.begin() + static_cast<long>(got));
      std::sort(v.begin(), v.end(), [](auto& a, auto& b) { return a.worker != b.worker ? a.worker < b.worker : a.ticket_ns < b.ticket_ns; });
      for (size_t i = 1; i < v.size(); ++i)
        if (v[i].worker == v[i - 1].worker) gaps.push_back((double)(int64_t)(v[i].ticket_ns - v[i - 1].ticket_ns) / 1e3);
      // fetcher cadence inside a batch (same worker, same ticket stamp):
      // seen -> first staged, and staged -> next staged (per-task handoff);
      // and across batches: last staged -> next batch's ticket
      std::vector<double> first_h, next_h, batch_gap, batch_n;
      for (size_t i = 0; i < v.size();) {
        size_t j = i;
        std::vector<uint64_t> deq;
        while (j < v.size() && v[j].worker == v[i].worker && v[j].ticket_ns == v[i].ticket_ns) deq.push_back(v[j++].dequeue_ns);
        std::sort(deq.begin(), deq.end());
        first_h.push_back((double)(int64_t)(deq[0] - v[i].seen_ns) / 1e3);
        for (size_t k = 1; k < deq.size(); ++k) next_h.push_back((double)(int64_t)(deq[k] - deq[k - 1]) / 1e3);
        batch_n.push_back((double)deq.size());
        if (j < v.size() && v[j].worker == v[i].worker) batch_gap.push_back((double)(int64_t)(v[j].ticket_ns - deq.back()) / 1e3);
        i = j;
      }
      auto med = [](std::vector<double> x, double q) {
        std::sort(x.begin(), x.end());
        return x.empty() ? 0.0 : x[static_cast<size_t>(q * (x.size() - 1))];
      };
      std::printf("  batch size mean %.2f | seen->first staged p50 %.2f p90 %.2f | staged->next staged p50 %.2f p90 %.2f"
                  " | last staged->next ticket p50 %.2f p90 %.2f us\n",
                  [&] { double t = 0; for (double x : batch_n) t += x; return batch_n.empty() ? 0.0 : t / batch_n.size(); }(),
                  med(first_h, .5), med(first_h, .9), med(next_h, .5), med(next_h, .9), med(batch_gap, .5), med(batch_gap, .9));
      std::sort(gaps.begin(), gaps.end());
      if (!gaps.empty())
        std::printf("  ticket gap per worker p50 %.2f us p90 %.2f us\n", gaps[gaps.size() / 2], gaps[gaps.size() * 9 / 10]);
    }
  }
  std::vector<float> got(total);
  rt.pool().download(Cv.buffer, got.data(), total * 4);
  int64_t bad = 0;
  for (int64_t i = 0; i < total; ++i)
    if (got[i] != ha[i] + hb[i]) ++bad;
  std::printf("mismatches %lld of %lld\n", (long long)bad, (long long)total);
  return bad != 0;
}
