// ref_bench.cpp — the reference CPU implementation timed on the host cores
// (bench.py cpu_baseline / --impl reference).  Drives the UNMODIFIED
// reference gpuos::Runtime (compiled from /root/reference/proj/include into
// oracle/_ref/ref_bench by oracle/Makefile) through its public API on the
// config-1 workload: N fp32 Add tasks of E elements with distinct a_i, b_i,
// c_i, worker pool = all hardware threads.
//
//   ref_bench --tasks N --elems E [--steps K | --seconds S]
// prints one JSON line: tasks_per_s, workers, tasks, seconds, step_seconds, p50_us
#include <gpuos/runtime.hpp>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace gpuos;

int main(int argc, char** argv) {
  int n = 10000, e = 4096, steps = 0;
  double seconds = 10.0;
  for (int i = 1; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--tasks")) n = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--elems")) e = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--steps")) steps = std::atoi(argv[i + 1]);
    else if (!std::strcmp(argv[i], "--seconds")) seconds = std::atof(argv[i + 1]);
  }
  RuntimeConfig cfg;
  cfg.workers.num_workers = std::thread::hardware_concurrency();
  Runtime rt(cfg);
  std::vector<TensorView> a, b, c;
  std::mt19937_64 rng(42 ^ (1 * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull));
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  for (int i = 0; i < n; ++i) {
    a.push_back(rt.alloc_tensor(DType::F32, {e}));
    b.push_back(rt.alloc_tensor(DType::F32, {e}));
    c.push_back(rt.alloc_tensor(DType::F32, {e}));
    float* pa = rt.pool().data<float>(a.back().buffer);
    float* pb = rt.pool().data<float>(b.back().buffer);
    for (int j = 0; j < e; ++j) pa[j] = static_cast<float>(dist(rng));
    for (int j = 0; j < e; ++j) pb[j] = static_cast<float>(dist(rng));
  }
  using clk = std::chrono::steady_clock;
  std::vector<double> step_s;
  const auto t_all = clk::now();
  for (int s = 0;; ++s) {
    if (steps > 0 && s >= steps) break;
    if (steps == 0 && s > 0 && std::chrono::duration<double>(clk::now() - t_all).count() >= seconds) break;
    const auto t0 = clk::now();
    for (int i = 0; i < n; ++i) rt.submit(OpKind::Add, {a[i], b[i]}, c[i]);
    rt.wait_all();
    step_s.push_back(std::chrono::duration<double>(clk::now() - t0).count());
  }
  // queue-depth-1 submit -> complete
  std::vector<double> lat;
  for (int i = 0; i < 2200; ++i) {
    const auto t0 = clk::now();
    TaskHandle h = rt.submit(OpKind::Add, {a[i % n], b[i % n]}, c[i % n]);
    rt.wait(h);
    if (i >= 200) lat.push_back(std::chrono::duration<double, std::micro>(clk::now() - t0).count());
  }
  std::sort(lat.begin(), lat.end());
  double tot = 0;
  for (double x : step_s) tot += x;
  std::printf("{\"tasks_per_s\": %.3f, \"workers\": %zu, \"tasks\": %llu, \"seconds\": %.4f, \"p50_us\": %.3f, "
              "\"step_seconds\": [",
              static_cast<double>(n) * static_cast<double>(step_s.size()) / tot, rt.num_workers(),
              static_cast<unsigned long long>(n) * step_s.size(), tot, lat[lat.size() / 2]);
  for (size_t i = 0; i < step_s.size(); ++i) std::printf("%s%.6f", i ? ", " : "", step_s[i]);
  std::printf("]}\n");
  return 0;
}
