// BASELINE.json configs 2-4 for bench.py (same library as gpuos_bench.cpp).
//
//   gb_config2: mixed micro-op stream: {Add, Mul, Relu,
//               ReduceSum} x {F32, F16, BF16, I32}, numel log-uniform in
//               [64, 65536], layouts contiguous / strided (stride-2, transposed
//               2-D) / broadcast ((1,C) row, rank-0 scalar); seed 42.
//   gb_config3: attention micro-ops, 32 heads x seq 128 x head_dim 64 as
//               individual tasks: Q*scale (rank-0), Q'.K^T (K as a transposed
//               view), row softmax, P.V; the host waits between the four
//               phases (the reference has no inter-task ordering).
//   gb_config4: operator hot swap under load: a stream of 4096-element fp32
//               tasks alternating the injected scale_add(1.5, -0.25) with
//               builtin Add; half way through, scale_add is re-injected at the
//               same id with (-2, 3) while the ring is full.
//
// Every config runs through gpuos::Runtime::submit; device time brackets the
// worker kernel's lifetime with CUDA events on its stream (as config 1).
#include <gpuos/runtime.hpp>
#include <immintrin.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace gpuos;

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
uint64_t config_seed(uint64_t seed, uint64_t config) {  // bench.hpp:280-282
  return seed ^ (config * 0x9e3779b97f4a7c15ull + 0x2545f4914f6cdd1dull);
}

struct Gen {  // one generated call of config 2 (operands inline: the stream is walked once, in order)
  OpKind op;
  struct In {
    TensorView v[2];
    int n = 0;
    void push_back(TensorView x) { v[n++] = std::move(x); }
  } in;
  TensorView out;
  double bytes;
  std::span<const TensorView> inputs() const { return std::span<const TensorView>(in.v, static_cast<size_t>(in.n)); }
};

TensorView view_of(const TensorView& base, int64_t offset, Shape shape, Strides strides) {
  TensorView v = base;
  v.offset = offset;
  v.shape = std::move(shape);
  v.strides = std::move(strides);
  return v;
}

// Narrowed doubles of the dtype, written through host staging + upload.
void fill_arena(Runtime& rt, const TensorView& t, int64_t n, DType dt, std::mt19937_64& rng) {
  std::uniform_real_distribution<double> u(-4.0, 4.0);
  std::uniform_int_distribution<int32_t> ui(-(1 << 14), (1 << 14) - 1);
  const size_t w = dtype_width(dt);
  std::vector<unsigned char> host(static_cast<size_t>(n) * w);
  for (int64_t i = 0; i < n; ++i) {
    switch (dt) {
      case DType::F32: {
        const float f = static_cast<float>(u(rng));
        std::memcpy(&host[i * 4], &f, 4);
        break;
      }
      case DType::I32: {
        const int32_t x = ui(rng);
        std::memcpy(&host[i * 4], &x, 4);
        break;
      }
      default: {  // f16 / bf16: any bit pattern of a finite value in range
        const float f = static_cast<float>(u(rng));
        uint32_t b;
        std::memcpy(&b, &f, 4);
        uint16_t h = 0;
        if (dt == DType::BF16) {
          h = static_cast<uint16_t>(b >> 16);
        } else {  // f16 by truncation of a value in [-4, 4)
          const uint32_t sign = (b >> 16) & 0x8000u;
          const int e = static_cast<int>((b >> 23) & 0xff) - 127 + 15;
          const uint32_t m = (b >> 13) & 0x3ffu;
          h = static_cast<uint16_t>(e <= 0 ? sign : (sign | (static_cast<uint32_t>(e) << 10) | m));
        }
        std::memcpy(&host[i * 2], &h, 2);
      }
    }
  }
  rt.pool().upload(t.buffer, host.data(), host.size());
}

struct Mixed {
  std::vector<Gen> calls;
  double bytes = 0;
};

// Config-2 stream over per-dtype arenas: inputs read from a shared input
// arena at random offsets, every output a distinct region.
Mixed make_mixed(Runtime& rt, int n_tasks, uint64_t seed) {
  const DType dts[4] = {DType::F32, DType::F16, DType::BF16, DType::I32};
  const OpKind ops[4] = {OpKind::Add, OpKind::Mul, OpKind::Relu, OpKind::ReduceSum};
  const int64_t kIn = int64_t{32} << 20;  // input elements per dtype (> L2 for every dtype)
  std::mt19937_64 rng(config_seed(seed, 2));
  std::uniform_real_distribution<double> lg(std::log(64.0), std::log(65536.0));
  std::uniform_int_distribution<int> pick4(0, 3), pick3(0, 2), pick2(0, 1);
  struct Plan {
    int op, dt, layout, sub;
    int64_t n, r, c;
  };
  std::vector<Plan> plans(static_cast<size_t>(n_tasks));
  int64_t out_need[4] = {0, 0, 0, 0};
  // GB_FORCE_{OP,DT,LAYOUT,SUB} pin one dimension of the distribution
  // (diagnostics: per-kind device cost)
  auto forced = [](const char* name) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : -1;
  };
  const int f_op = forced("GB_FORCE_OP"), f_dt = forced("GB_FORCE_DT"), f_lay = forced("GB_FORCE_LAYOUT"),
            f_sub = forced("GB_FORCE_SUB");
  for (Plan& p : plans) {
    p.op = pick4(rng);
    p.dt = pick4(rng);
    p.n = static_cast<int64_t>(std::llround(std::exp(lg(rng))));
    p.layout = pick3(rng);
    p.sub = pick2(rng);
    if (f_op >= 0) p.op = f_op;
    if (f_dt >= 0) p.dt = f_dt;
    if (f_lay >= 0) p.layout = f_lay;
    if (f_sub >= 0) p.sub = f_sub;
    // a 2-D factorisation R x C ~ n with R a power of two
    int64_t r = 1;
    while (r * r * 4 < p.n) r <<= 1;
    p.r = r;
    p.c = std::max<int64_t>(1, p.n / r);
    if (p.op == 3 || p.layout != 0) p.n = p.r * p.c;
    out_need[p.dt] += p.op == 3 ? p.r : p.n;
  }
  Mixed m;
  std::vector<TensorView> inA(4), outA(4);
  for (int d = 0; d < 4; ++d) {
    inA[d] = rt.alloc_tensor(dts[d], {kIn});
    fill_arena(rt, inA[d], kIn, dts[d], rng);
    outA[d] = rt.alloc_tensor(dts[d], {std::max<int64_t>(out_need[d], 1)});
  }
  int64_t out_cur[4] = {0, 0, 0, 0};
  std::uniform_int_distribution<int64_t> off(0, kIn - 2 * 65536 - 16);
  for (const Plan& p : plans) {
    Gen g;
    g.op = ops[p.op];
    const DType dt = dts[p.dt];
    const double w = static_cast<double>(dtype_width(dt));
    const TensorView& IN = inA[p.dt];
    const TensorView& OUT = outA[p.dt];
    const int arity = (g.op == OpKind::Relu || g.op == OpKind::ReduceSum) ? 1 : 2;
    const int64_t R = p.r, Cc = p.c, n = p.n;
    if (g.op == OpKind::ReduceSum) {
      // last-axis reduction of a 2-D (R, C) view: contiguous or transposed
      g.out = view_of(OUT, out_cur[p.dt], {R}, {1});
      out_cur[p.dt] += R;
      if (p.layout == 1) g.in.push_back(view_of(IN, off(rng), {R, Cc}, {1, R}));
      else g.in.push_back(view_of(IN, off(rng), {R, Cc}, {Cc, 1}));
      g.bytes = (static_cast<double>(R * Cc) + static_cast<double>(R)) * w;
    } else if (p.layout == 0) {  // contiguous
      g.out = view_of(OUT, out_cur[p.dt], {n}, {1});
      out_cur[p.dt] += n;
      for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {n}, {1}));
      g.bytes = static_cast<double>(n) * w * (arity + 1);
    } else if (p.layout == 1) {  // strided: stride-2 of a 2x span, or a transposed 2-D view
      if (p.sub == 0) {
        g.out = view_of(OUT, out_cur[p.dt], {n}, {1});
        for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {n}, {2}));
      } else {
        g.out = view_of(OUT, out_cur[p.dt], {R, Cc}, {Cc, 1});
        for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {R, Cc}, {1, R}));
      }
      out_cur[p.dt] += n;
      g.bytes = static_cast<double>(n) * w * (arity + 1);
    } else {  // broadcast: a (1, C) row against (R, C), or a rank-0 scalar
      g.out = view_of(OUT, out_cur[p.dt], {R, Cc}, {Cc, 1});
      out_cur[p.dt] += n;
      double src = 0;
      if (arity == 1) {
        if (p.sub == 0) {
          g.in.push_back(view_of(IN, off(rng), {1, Cc}, {Cc, 1}));
          src = static_cast<double>(Cc);
        } else {
          g.in.push_back(view_of(IN, off(rng), {}, {}));
          src = 1;
        }
      } else {
        g.in.push_back(view_of(IN, off(rng), {R, Cc}, {Cc, 1}));
        if (p.sub == 0) {
          g.in.push_back(view_of(IN, off(rng), {1, Cc}, {Cc, 1}));
          src = static_cast<double>(n + Cc);
        } else {
          g.in.push_back(view_of(IN, off(rng), {}, {}));
          src = static_cast<double>(n + 1);
        }
      }
      g.bytes = (src + static_cast<double>(n)) * w;
    }
    m.bytes += g.bytes;
    m.calls.push_back(std::move(g));
  }
  return m;
}

struct Events {
  gpuos_dev* dev;
  void* e0 = nullptr;
  void* e1 = nullptr;
  void* ks = nullptr;
  explicit Events(gpuos_dev* d) : dev(d) {
    check_abi(gpuos_event_create(dev, &e0), "ev");
    check_abi(gpuos_event_create(dev, &e1), "ev");
    check_abi(gpuos_dev_kernel_stream(dev, &ks), "ks");
  }
  ~Events() {
    gpuos_event_destroy(dev, e0);
    gpuos_event_destroy(dev, e1);
  }
  // one worker-kernel lifetime around `body`; returns device ms
  template <class F>
  double generation(F body) {
    check_abi(gpuos_event_record(dev, e0, ks), "ev0");
    check_abi(gpuos_dev_start(dev), "start");
    check_abi(gpuos_event_record(dev, e1, ks), "ev1");
    body();
    check_abi(gpuos_dev_stop(dev), "stop");
    check_abi(gpuos_event_sync(dev, e1), "sync");
    float ms = 0;
    check_abi(gpuos_event_elapsed_ms(dev, e0, e1, &ms), "elapsed");
    return ms;
  }
};

RuntimeConfig bench_cfg(int device, size_t capacity) {
  RuntimeConfig cfg;
  cfg.device = device;
  cfg.capacity = capacity;
  cfg.telemetry_enabled = false;
  cfg.device_buffers = true;
  if (const char* w = std::getenv("GB_WORKERS")) cfg.workers.num_workers = static_cast<size_t>(std::atoi(w));
  return cfg;
}

}  // namespace

extern "C" {

// out: [0] tasks/s (device), [1] algorithmic GB/s, [2] tasks per step,
//      [3] mean bytes/task, [4] failed tasks, [5] host submit ns/task
int gb_config2(int device, int n_tasks, int steps, double* out) {
  Runtime rt(bench_cfg(device, 4096));
  Mixed m = make_mixed(rt, n_tasks, 42);
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  Events ev(rt.device());
  std::vector<TaskHandle> hs;
  hs.reserve(m.calls.size());
  double dev_ms = 0, sub_ms = 0;
  uint64_t failed = 0;
  for (int s = 0; s < steps + 1; ++s) {  // step 0 warms up
    hs.clear();
    double t_sub = 0;
    const double ms = ev.generation([&] {
      const double t0 = now_ms();
      for (const Gen& g : m.calls)
        hs.push_back(rt.submit_span(static_cast<uint64_t>(g.op), g.inputs(), g.out, std::span<const double>()));
      t_sub = now_ms() - t0;
      rt.wait_all();
    });
    if (s == 0) continue;
    dev_ms += ms;
    sub_ms += t_sub;
    for (const TaskHandle& h : hs) failed += h.state() == TaskState::Failed ? 1 : 0;
  }
  const double tasks = static_cast<double>(m.calls.size()) * steps;
  out[0] = tasks / (dev_ms / 1e3);
  out[1] = m.bytes * steps / (dev_ms / 1e3) / 1e9;
  out[2] = static_cast<double>(m.calls.size());
  out[3] = m.bytes / static_cast<double>(m.calls.size());
  out[4] = static_cast<double>(failed);
  out[5] = sub_ms * 1e6 / tasks;
  return 0;
}

// out: [0] step us (median), [1] tasks/s, [2] GFLOP/s, [3] failed tasks,
//      [4] max |o - ref| / max(1,|ref|) over head 0 (fp64 host reference),
//      [5..8] median us of the scale / QK^T / softmax / PV phases
int gb_config3(int device, int dtype, int steps, double* out) {
  const int H = 32, S = 128, D = 64;
  const DType dt = static_cast<DType>(dtype);
  Runtime rt(bench_cfg(device, 4096));
  TensorView Q = rt.alloc_tensor(dt, {H, S, D}), K = rt.alloc_tensor(dt, {H, S, D}), V = rt.alloc_tensor(dt, {H, S, D});
  TensorView Qs = rt.alloc_tensor(dt, {H, S, D}), Sc = rt.alloc_tensor(dt, {H, S, S}), P = rt.alloc_tensor(dt, {H, S, S});
  TensorView O = rt.alloc_tensor(dt, {H, S, D}), scale = rt.alloc_tensor(dt, {1});
  std::mt19937_64 rng(config_seed(42, 3));
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  auto narrow = [&](double x) -> double {
    if (dt == DType::F32) return static_cast<double>(static_cast<float>(x));
    float f = static_cast<float>(x);  // bf16: round to nearest even on the top 16 bits
    uint32_t b;
    std::memcpy(&b, &f, 4);
    b = (b + 0x7fffu + ((b >> 16) & 1u)) & 0xffff0000u;
    std::memcpy(&f, &b, 4);
    return f;
  };
  const size_t nq = static_cast<size_t>(H) * S * D;
  std::vector<double> q(nq), k(nq), v(nq);
  for (auto* vec : {&q, &k, &v})
    for (double& x : *vec) x = narrow(u(rng));
  auto upload = [&](const TensorView& t, const std::vector<double>& vals) {
    if (dt == DType::F32) {
      std::vector<float> f(vals.begin(), vals.end());
      rt.pool().upload(t.buffer, f.data(), f.size() * 4);
    } else {
      std::vector<uint16_t> b(vals.size());
      for (size_t i = 0; i < vals.size(); ++i) {
        const float f = static_cast<float>(vals[i]);
        uint32_t x;
        std::memcpy(&x, &f, 4);
        b[i] = static_cast<uint16_t>(x >> 16);
      }
      rt.pool().upload(t.buffer, b.data(), b.size() * 2);
    }
  };
  upload(Q, q);
  upload(K, k);
  upload(V, v);
  upload(scale, {0.125});
  auto head = [&](const TensorView& t, int h, int64_t rows, int64_t cols) {
    return view_of(t, static_cast<int64_t>(h) * rows * cols, {rows, cols}, {cols, 1});
  };
  const TensorView sc0 = view_of(scale, 0, {}, {});
  std::vector<double> step_us;
  std::vector<double> phase_us[4];
  uint64_t failed = 0;
  std::vector<TaskHandle> hs;
  for (int s = 0; s < steps + 2; ++s) {
    const double t0 = now_ms();
    for (int phase = 0; phase < 4; ++phase) {
      const double tp = now_ms();
      hs.clear();
      for (int h = 0; h < H; ++h) {
        switch (phase) {
          case 0: hs.push_back(rt.submit(OpKind::Mul, {head(Q, h, S, D), sc0}, head(Qs, h, S, D))); break;
          case 1: {  // K^T as a transposed view: shape (D, S), strides (1, D)
            const TensorView kt = view_of(K, static_cast<int64_t>(h) * S * D, {D, S}, {1, D});
            hs.push_back(rt.submit(OpKind::MatMulSmall, {head(Qs, h, S, D), kt}, head(Sc, h, S, S)));
            break;
          }
          case 2: hs.push_back(rt.submit(OpKind::Softmax, {head(Sc, h, S, S)}, head(P, h, S, S))); break;
          default: hs.push_back(rt.submit(OpKind::MatMulSmall, {head(P, h, S, S), head(V, h, S, D)}, head(O, h, S, D)));
        }
      }
      for (const TaskHandle& th : hs) {
        th.wait();
        if (s >= 2) failed += th.state() == TaskState::Failed ? 1 : 0;
      }
      if (s >= 2) phase_us[phase].push_back((now_ms() - tp) * 1e3);
    }
    if (s >= 2) step_us.push_back((now_ms() - t0) * 1e3);
  }
  std::sort(step_us.begin(), step_us.end());
  const double med = step_us[step_us.size() / 2];
  // fp64 reference for head 0 from the narrowed inputs
  std::vector<double> o(static_cast<size_t>(S) * D);
  {
    std::vector<double> sc(static_cast<size_t>(S) * S);
    for (int i = 0; i < S; ++i) {
      double mx = -1e300;
      for (int j = 0; j < S; ++j) {
        double acc = 0;
        for (int d = 0; d < D; ++d) acc += narrow(q[i * D + d] * 0.125) * k[j * D + d];
        sc[i * S + j] = narrow(acc);
        mx = std::max(mx, sc[i * S + j]);
      }
      double den = 0;
      for (int j = 0; j < S; ++j) den += std::exp(sc[i * S + j] - mx);
      for (int j = 0; j < S; ++j) sc[i * S + j] = narrow(std::exp(sc[i * S + j] - mx) / den);
    }
    for (int i = 0; i < S; ++i)
      for (int d = 0; d < D; ++d) {
        double acc = 0;
        for (int j = 0; j < S; ++j) acc += sc[i * S + j] * v[j * D + d];
        o[i * D + d] = narrow(acc);
      }
  }
  std::vector<double> got(static_cast<size_t>(S) * D);
  if (dt == DType::F32) {
    std::vector<float> f(got.size());
    rt.pool().download(O.buffer, f.data(), f.size() * 4);
    for (size_t i = 0; i < f.size(); ++i) got[i] = f[i];
  } else {
    std::vector<uint16_t> b(got.size());
    rt.pool().download(O.buffer, b.data(), b.size() * 2);
    for (size_t i = 0; i < b.size(); ++i) {
      const uint32_t x = static_cast<uint32_t>(b[i]) << 16;
      float f;
      std::memcpy(&f, &x, 4);
      got[i] = f;
    }
  }
  double err = 0;
  for (size_t i = 0; i < got.size(); ++i) err = std::max(err, std::fabs(got[i] - o[i]) / std::max(1.0, std::fabs(o[i])));
  const double flops = 2.0 * H * (2.0 * S * S * D);  // QK^T + PV
  out[0] = med;
  out[1] = 4.0 * H / (med / 1e6);
  out[2] = flops / (med / 1e6) / 1e9;
  out[3] = static_cast<double>(failed);
  out[4] = err;
  for (int ph = 0; ph < 4; ++ph) {  // [5..8] median us of scale / QK^T / softmax / PV phases
    std::sort(phase_us[ph].begin(), phase_us[ph].end());
    out[5 + ph] = phase_us[ph][phase_us[ph].size() / 2];
  }
  return 0;
}

// out: [0] tasks/s (device), [1] inject call ms (template compile + install),
//      [2] upload us, [3] epoch wait us, [4] bank write us, [5] flip us,
//      [6] checked rows, [7] rows not uniformly one variant, [8] rows with the
//      old variant after the swap window, [9] failed tasks, [10] canary hits,
//      [11] old rows, [12] new rows
int gb_config4(int device, int n_tasks, double* out) {
  const int64_t E = 4096;
  const int kIn = 8;
  const int kWin = 16384;  // tasks each side of the swap keep a dedicated output row
  const int kRR = 8192;    // the rest share rows round robin (>> tasks in flight)
  Runtime rt(bench_cfg(device, 4096));
  const double pa[2] = {1.5, -0.25}, pb[2] = {-2.0, 3.0};
  const uint32_t id = static_cast<uint32_t>(rt.inject_operator("scale_add", pa));
  TensorView IN = rt.alloc_tensor(DType::F32, {kIn * E});
  TensorView OUT = rt.alloc_tensor(DType::F32, {int64_t{2 * kWin + kRR} * E});
  std::vector<float> x(static_cast<size_t>(kIn * E));
  std::mt19937_64 rng(config_seed(42, 4));
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (float& f : x) f = static_cast<float>(u(rng));
  rt.pool().upload(IN.buffer, x.data(), x.size() * 4);
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  Events ev(rt.device());
  std::vector<int> variant(static_cast<size_t>(n_tasks), 0);  // 0 add, 1 scale_add
  double inject_ms = 0;
  gpuos_inject_stats st{};
  std::vector<TaskHandle> hs;
  hs.reserve(static_cast<size_t>(n_tasks));
  const int swap_at = n_tasks / 2;
  auto row_of = [&](int t) -> int64_t {
    if (t >= swap_at - kWin && t < swap_at + kWin) return t - (swap_at - kWin);
    return 2 * kWin + t % kRR;
  };
  const double ms = ev.generation([&] {
    for (int t = 0; t < n_tasks; ++t) {
      const TensorView in = view_of(IN, static_cast<int64_t>(t % kIn) * E, {E}, {1});
      const TensorView o = view_of(OUT, row_of(t) * E, {E}, {1});
      if (t % 2 == 0) {
        hs.push_back(rt.submit(OpKind::Add, {in, in}, o));
      } else {
        hs.push_back(rt.submit(static_cast<uint64_t>(id), {in}, o));
        variant[static_cast<size_t>(t)] = 1;
      }
      if (t == swap_at) {
        const double t0 = now_ms();
        rt.inject_operator_at(id, "scale_add", pb);
        inject_ms = now_ms() - t0;
        st = rt.last_inject_stats();
      }
    }
    rt.wait_all();
  });
  // the window around the swap: every row entirely one variant (one bank per
  // dispatch, test_executor.cpp:330-387); past the ring's in-flight window
  // only the new variant may appear
  std::vector<float> got(static_cast<size_t>(2 * kWin) * E);
  rt.pool().download(OUT.buffer, got.data(), got.size() * 4);
  uint64_t checked = 0, mixed = 0, late_old = 0, old_rows = 0, new_rows = 0, failed = 0;
  for (const TaskHandle& h : hs) failed += h.state() == TaskState::Failed ? 1 : 0;
  for (int t = std::max(0, swap_at - kWin); t < std::min(n_tasks, swap_at + kWin); ++t) {
    const float* row = &got[static_cast<size_t>(row_of(t)) * E];
    const float* xin = &x[static_cast<size_t>(t % kIn) * E];
    ++checked;
    if (variant[static_cast<size_t>(t)] == 0) {
      bool ok = true;
      for (int64_t e = 0; e < E; ++e) ok = ok && row[e] == xin[e] + xin[e];
      mixed += ok ? 0 : 1;
      continue;
    }
    bool all_a = true, all_b = true;
    for (int64_t e = 0; e < E; ++e) {
      const double xv = xin[e];
      all_a = all_a && row[e] == static_cast<float>(xv * 1.5 + -0.25);
      all_b = all_b && row[e] == static_cast<float>(xv * -2.0 + 3.0);
    }
    if (!all_a && !all_b) ++mixed;
    if (all_a) ++old_rows;
    if (all_b) ++new_rows;
    if (all_a && !all_b && t > swap_at + 4096) ++late_old;
  }
  out[0] = n_tasks / (ms / 1e3);
  out[1] = inject_ms;
  out[2] = st.upload_ns / 1e3;
  out[3] = st.epoch_wait_ns / 1e3;
  out[4] = st.bank_write_ns / 1e3;
  out[5] = st.flip_ns / 1e3;
  out[6] = static_cast<double>(checked);
  out[7] = static_cast<double>(mixed);
  out[8] = static_cast<double>(late_old);
  out[9] = static_cast<double>(failed);
  out[10] = static_cast<double>(rt.canary_hits());
  out[11] = static_cast<double>(old_rows);
  out[12] = static_cast<double>(new_rows);
  return 0;
}

// Native promotion of an injected operator (config 4, second half): a stream
// of 4096-element fp32 scale_add tasks run as a device program, then the op
// is promoted to native code (NVRTC + nvJitLink + generation handover) and
// the same stream runs again.
// out: [0] program tasks/s, [1] native tasks/s, [2] codegen ms, [3] nvrtc ms,
//      [4] nvJitLink ms, [5] drain us, [6] module load us, [7] relaunch us,
//      [8] table flip us, [9] output mismatches native vs program
int gb_native(int device, int n_tasks, double* out) {
  const int64_t E = 4096;
  const int kRows = 2048;
  Runtime rt(bench_cfg(device, 4096));
  const double pa[2] = {1.5, -0.25};
  const uint32_t id = static_cast<uint32_t>(rt.inject_operator("scale_add", pa));
  TensorView IN = rt.alloc_tensor(DType::F32, {int64_t{kRows} * E});
  TensorView OA = rt.alloc_tensor(DType::F32, {int64_t{kRows} * E});
  TensorView OB = rt.alloc_tensor(DType::F32, {int64_t{kRows} * E});
  std::vector<float> x(static_cast<size_t>(kRows) * E);
  std::mt19937_64 rng(config_seed(42, 4));
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (float& f : x) f = static_cast<float>(u(rng));
  rt.pool().upload(IN.buffer, x.data(), x.size() * 4);
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  Events ev(rt.device());
  auto stream = [&](const TensorView& O) {
    return ev.generation([&] {
      for (int t = 0; t < n_tasks; ++t) {
        const int64_t r = t % kRows;
        rt.submit(static_cast<uint64_t>(id), {view_of(IN, r * E, {E}, {1})}, view_of(O, r * E, {E}, {1}));
      }
      rt.wait_all();
    });
  };
  stream(OA);  // warm
  const double ms_prog = stream(OA);
  rt.promote_native(id);  // workers stopped: the handover only loads + records the module
  const auto& st = rt.last_native_stats();
  stream(OB);  // warm
  const double ms_nat = stream(OB);
  std::vector<float> a(x.size()), b(x.size());
  rt.pool().download(OA.buffer, a.data(), a.size() * 4);
  rt.pool().download(OB.buffer, b.data(), b.size() * 4);
  uint64_t bad = 0;
  for (size_t i = 0; i < a.size(); ++i) bad += std::memcmp(&a[i], &b[i], 4) != 0;
  out[0] = n_tasks / (ms_prog / 1e3);
  out[1] = n_tasks / (ms_nat / 1e3);
  out[2] = st.codegen_ns / 1e6;
  out[3] = st.compile_ns / 1e6;
  out[4] = st.link_ns / 1e6;
  out[5] = st.handover.drain_ns / 1e3;
  out[6] = st.handover.load_ns / 1e3;
  out[7] = st.handover.relaunch_ns / 1e3;
  out[8] = (st.install.upload_ns + st.install.epoch_wait_ns + st.install.bank_write_ns + st.install.flip_ns) / 1e3;
  out[9] = static_cast<double>(bad);
  return 0;
}

// Config 5 on one GPU: `streams` independent task streams (config-2
// distribution, seeds 42+s), each from its own host producer thread into its
// own runtime (ring + persistent generation of `workers` CTAs: the streams
// split the SMs), all on `device`.  On G GPUs the same streams shard s -> s%G
// (bench.py --gpus G runs one replica per GPU).
// out: [0] aggregate tasks/s (all streams / slowest stream's device time),
//      [1] aggregate algorithmic GB/s, [2] failed tasks, [3] slowest stream ms
int gb_config5(int device, int streams, int tasks_per_stream, int workers, double* out) {
  struct Stream {
    std::unique_ptr<Runtime> rt;
    Mixed m;
    double ms = 0;
    uint64_t failed = 0;
  };
  std::vector<Stream> ss(static_cast<size_t>(streams));
  for (int i = 0; i < streams; ++i) {
    RuntimeConfig cfg = bench_cfg(device, 4096);
    cfg.workers.num_workers = static_cast<size_t>(workers);
    ss[static_cast<size_t>(i)].rt = std::make_unique<Runtime>(cfg);
    ss[static_cast<size_t>(i)].m = make_mixed(*ss[static_cast<size_t>(i)].rt, tasks_per_stream, 42 + static_cast<uint64_t>(i));
    ss[static_cast<size_t>(i)].rt->wait_all();
  }
  auto run = [&](Stream& st) {
    Runtime& rt = *st.rt;
    std::vector<TaskHandle> hs;
    hs.reserve(st.m.calls.size());
    void *e0 = nullptr, *e1 = nullptr, *ks = nullptr;
    check_abi(gpuos_event_create(rt.device(), &e0), "ev");
    check_abi(gpuos_event_create(rt.device(), &e1), "ev");
    check_abi(gpuos_dev_kernel_stream(rt.device(), &ks), "ks");
    check_abi(gpuos_dev_stop(rt.device()), "stop");
    check_abi(gpuos_event_record(rt.device(), e0, ks), "ev0");
    check_abi(gpuos_dev_start(rt.device()), "start");
    check_abi(gpuos_event_record(rt.device(), e1, ks), "ev1");
    for (const Gen& g : st.m.calls)
      hs.push_back(rt.submit_span(static_cast<uint64_t>(g.op), g.inputs(), g.out, std::span<const double>()));
    rt.wait_all();
    check_abi(gpuos_dev_stop(rt.device()), "stop");
    check_abi(gpuos_event_sync(rt.device(), e1), "sync");
    float ms = 0;
    check_abi(gpuos_event_elapsed_ms(rt.device(), e0, e1, &ms), "elapsed");
    st.ms = ms;
    for (const TaskHandle& h : hs) st.failed += h.state() == TaskState::Failed ? 1 : 0;
    gpuos_event_destroy(rt.device(), e0);
    gpuos_event_destroy(rt.device(), e1);
    check_abi(gpuos_dev_start(rt.device()), "restart");
  };
  for (Stream& st : ss) run(st);  // warm each stream alone
  std::vector<std::thread> th;
  for (Stream& st : ss) th.emplace_back([&run, &st] { run(st); });
  for (std::thread& t : th) t.join();
  double slow = 0, bytes = 0;
  uint64_t failed = 0, tasks = 0;
  for (const Stream& st : ss) {
    slow = std::max(slow, st.ms);
    bytes += st.m.bytes;
    failed += st.failed;
    tasks += st.m.calls.size();
  }
  out[0] = static_cast<double>(tasks) / (slow / 1e3);
  out[1] = bytes / (slow / 1e3) / 1e9;
  out[2] = static_cast<double>(failed);
  out[3] = slow;
  return 0;
}

}  // extern "C"
