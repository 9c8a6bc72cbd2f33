// Burst-after-idle timeline (config 3's phase shape): the runtime idles, then
// 32 tasks (Q * scale, 128 x 64 f32 each, a rank-0 broadcast: extended slots)
// are submitted back to back and waited; per task: enqueue -> seen -> dequeue
// -> end -> done from the device trace, relative to the first enqueue.
//   build/probe/burst_probe [bursts=5] [idle_us=1000]
#include <gpuos/runtime.hpp>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

using namespace gpuos;

int main(int argc, char** argv) {
  const int bursts = argc > 1 ? std::atoi(argv[1]) : 5;
  const int idle_us = argc > 2 ? std::atoi(argv[2]) : 1000;
  RuntimeConfig cfg;
  cfg.telemetry_enabled = true;
  cfg.trace_capacity = 4096;
  Runtime rt(cfg);
  const int H = 32, S = 128, D = 64;
  TensorView Q = rt.alloc_tensor(DType::F32, {H, S, D}), Qs = rt.alloc_tensor(DType::F32, {H, S, D});
  TensorView sc = rt.alloc_tensor(DType::F32, {1});
  TensorView s0 = sc;
  s0.shape = {};
  s0.strides = {};
  for (int b = 0; b < bursts; ++b) {
    std::this_thread::sleep_for(std::chrono::microseconds(idle_us));
    std::vector<TaskHandle> hs;
    const uint64_t t0 = monotonic_ns();
    for (int h = 0; h < H; ++h) {
      TensorView q = Q, o = Qs;
      q.shape = o.shape = {S, D};
      q.strides = o.strides = {D, 1};
      q.offset = o.offset = int64_t{h} * S * D;
      const int kind = std::getenv("BURST_KIND") ? std::atoi(std::getenv("BURST_KIND")) : 0;
      if (kind == 0) hs.push_back(rt.submit(OpKind::Mul, {q, s0}, o));       // rank-0 broadcast (extended slot)
      else if (kind == 1) hs.push_back(rt.submit(OpKind::Mul, {q, q}, o));   // dense (compact slot)
      else hs.push_back(rt.submit(OpKind::Relu, {q}, o));                    // dense unary (compact slot)
    }
    const uint64_t t_sub = monotonic_ns();
    for (const TaskHandle& th : hs) th.wait();
    const uint64_t t_done = monotonic_ns();
    std::vector<gpuos_trace_phase> ph(4096);
    uint64_t n = 0;
    gpuos_trace_phases(rt.device(), ph.data(), ph.size(), &n);
    std::vector<gpuos_trace_phase> mine;
    for (uint64_t i = 0; i < n; ++i)
      if (ph[i].seq >= hs.front().id() && ph[i].seq <= hs.back().id()) mine.push_back(ph[i]);
    std::sort(mine.begin(), mine.end(), [](auto& a, auto& x) { return a.seq < x.seq; });
    auto us = [&](uint64_t t) { return (double)(int64_t)(t - t0) / 1e3; };
    std::vector<double> seen, deq, end, done;
    for (auto& p : mine) {
      seen.push_back(us(p.seen_ns));
      deq.push_back(us(p.dequeue_ns));
      end.push_back(us(p.end_ns));
      done.push_back(us(p.done_ns));
    }
    auto mm = [](std::vector<double> v) {
      std::sort(v.begin(), v.end());
      return v.empty() ? std::make_pair(0.0, 0.0) : std::make_pair(v.front(), v.back());
    };
    if (b == bursts - 1 && std::getenv("BURST_DETAIL")) {
      std::sort(mine.begin(), mine.end(), [](auto& x, auto& y) { return x.seen_ns < y.seen_ns; });
      for (auto& p : mine)
        std::printf("  seq %llu worker %u ticket %.1f seen %.1f deq %.1f end %.1f done %.1f\n", (unsigned long long)p.seq,
                    p.worker, us(p.ticket_ns), us(p.seen_ns), us(p.dequeue_ns), us(p.end_ns), us(p.done_ns));
    }
    const auto a = mm(seen), d = mm(deq), e = mm(end), f = mm(done);
    std::printf("burst %d: %zu traced | submit %.1f us | seen %.1f..%.1f | deq %.1f..%.1f | end %.1f..%.1f | done "
                "%.1f..%.1f | host waited %.1f us\n",
                b, mine.size(), (t_sub - t0) / 1e3, a.first, a.second, d.first, d.second, e.first, e.second, f.first,
                f.second, (t_done - t0) / 1e3);
  }
  return 0;
}
