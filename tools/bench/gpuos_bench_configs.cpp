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

#include "oracle_check.hpp"

#include <algorithm>
#include <atomic>
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

// Input arenas: F32, F16, BF16, I32 for mul/relu/sum (U[-2^15, 2^15)) and
// I32 for add (U[-2^30, 2^30)), so the oracle never overflows.
enum Arena { kAF32 = 0, kAF16, kABF16, kAI32S, kAI32B, kArenas };

struct Gen {  // one generated call of config 2 (operands inline: the stream is walked once, in order)
  OpKind op;
  struct In {
    TensorView v[2];
    int n = 0;
    void push_back(TensorView x) { v[n++] = std::move(x); }
  } in;
  TensorView out;
  double bytes;
  uint8_t dt;         // 0 F32, 1 F16, 2 BF16, 3 I32 (output arena index)
  uint8_t arena;      // input arena
  bool survives;      // output not overwritten later in the stream (output-ring wrap)
  std::span<const TensorView> inputs() const { return std::span<const TensorView>(in.v, static_cast<size_t>(in.n)); }
};

TensorView view_of(const TensorView& base, int64_t offset, Shape shape, Strides strides) {
  TensorView v = base;
  v.offset = offset;
  v.shape = std::move(shape);
  v.strides = std::move(strides);
  return v;
}

// Narrowed doubles of the dtype, kept on the host (the checker's copy) and uploaded.
void fill_arena(Runtime& rt, const TensorView& t, int64_t n, int arena, std::mt19937_64& rng,
                std::vector<unsigned char>& host) {
  std::uniform_real_distribution<double> u(-4.0, 4.0);
  std::uniform_int_distribution<int32_t> us(-(1 << 15), (1 << 15) - 1), ub(-(1 << 30), (1 << 30) - 1);
  const bool i32 = arena == kAI32S || arena == kAI32B;
  const size_t w = (arena == kAF16 || arena == kABF16) ? 2 : 4;
  host.resize(static_cast<size_t>(n) * w);
  for (int64_t i = 0; i < n; ++i) {
    if (i32) {
      const int32_t x = arena == kAI32S ? us(rng) : ub(rng);
      std::memcpy(&host[i * 4], &x, 4);
    } else if (arena == kAF32) {
      const float f = static_cast<float>(u(rng));
      std::memcpy(&host[i * 4], &f, 4);
    } else {  // f16 / bf16: any bit pattern of a finite value in range
      const float f = static_cast<float>(u(rng));
      uint32_t b;
      std::memcpy(&b, &f, 4);
      uint16_t h = 0;
      if (arena == kABF16) {
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
  rt.pool().upload(t.buffer, host.data(), host.size());
}

struct Mixed {
  std::vector<Gen> calls;
  double bytes = 0;
  TensorView inA[kArenas];
  std::vector<unsigned char> host_in[kArenas];  // the checker's copy of every input arena
  TensorView outA[4];
  int64_t out_len[4] = {0, 0, 0, 0};
  uint64_t survivors = 0;
};

// Config-2 stream: ops and dtypes uniform, numel log-uniform
// in [64, 65536], layouts 1/3 each; inputs read from shared per-dtype arenas
// at random offsets.  Outputs are carved in order from one output arena per
// dtype.  `out_cap` > 0 makes that arena a ring of out_cap elements (long
// multi-stream runs): a region is then reused only after out_cap later
// output elements of its dtype -- tens of thousands of tasks, far beyond the
// ring capacity plus the tasks executing -- so no two in-flight tasks ever
// share output memory; only the last lap's outputs survive to be checked.
Mixed make_mixed(Runtime& rt, int n_tasks, uint64_t seed, int64_t out_cap = 0) {
  const DType dts[4] = {DType::F32, DType::F16, DType::BF16, DType::I32};
  const OpKind ops[4] = {OpKind::Add, OpKind::Mul, OpKind::Relu, OpKind::ReduceSum};
  const int64_t kIn = int64_t{32} << 20;  // input elements per arena (> L2 for every dtype)
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
  for (int a = 0; a < kArenas; ++a) {
    const DType dt = a == kAF32 ? DType::F32 : a == kAF16 ? DType::F16 : a == kABF16 ? DType::BF16 : DType::I32;
    m.inA[a] = rt.alloc_tensor(dt, {kIn});
    fill_arena(rt, m.inA[a], kIn, a, rng, m.host_in[a]);
  }
  int64_t cap[4];
  for (int d = 0; d < 4; ++d) {
    cap[d] = std::max<int64_t>(out_cap > 0 ? std::min(out_cap, out_need[d]) : out_need[d], 65536);
    m.out_len[d] = cap[d];
    m.outA[d] = rt.alloc_tensor(dts[d], {cap[d]});
  }
  int64_t tot[4] = {0, 0, 0, 0};  // unwrapped output cursor per dtype
  std::vector<int64_t> start(plans.size());
  m.calls.reserve(plans.size());
  std::uniform_int_distribution<int64_t> off_raw(0, kIn - 2 * 65536 - 16);
  // GB_FORCE_ALIGN=1 (diagnostics): every view starts 16-byte aligned
  const bool align16 = std::getenv("GB_FORCE_ALIGN") != nullptr;
  auto off = [&](std::mt19937_64& r) { return align16 ? off_raw(r) & ~int64_t{7} : off_raw(r); };
  for (size_t pi = 0; pi < plans.size(); ++pi) {
    const Plan& p = plans[pi];
    Gen g;
    g.op = ops[p.op];
    g.dt = static_cast<uint8_t>(p.dt);
    const DType dt = dts[p.dt];
    const double w = static_cast<double>(dtype_width(dt));
    const int arity = (g.op == OpKind::Relu || g.op == OpKind::ReduceSum) ? 1 : 2;
    g.arena = static_cast<uint8_t>(p.dt < 3 ? p.dt : (g.op == OpKind::Add ? kAI32B : kAI32S));
    const TensorView& IN = m.inA[g.arena];
    const TensorView& OUT = m.outA[p.dt];
    const int64_t R = p.r, Cc = p.c, n = p.n;
    const int64_t n_out = g.op == OpKind::ReduceSum ? R : n;
    if (align16) tot[p.dt] = (tot[p.dt] + 7) & ~int64_t{7};
    int64_t pos = tot[p.dt] % cap[p.dt];
    if (pos + n_out > cap[p.dt]) {  // next lap
      tot[p.dt] += cap[p.dt] - pos;
      pos = 0;
    }
    start[pi] = tot[p.dt];
    tot[p.dt] += n_out;
    const int64_t o = pos;
    if (g.op == OpKind::ReduceSum) {
      // last-axis reduction of a 2-D (R, C) view: contiguous or transposed
      g.out = view_of(OUT, o, {R}, {1});
      if (p.layout == 1) g.in.push_back(view_of(IN, off(rng), {R, Cc}, {1, R}));
      else g.in.push_back(view_of(IN, off(rng), {R, Cc}, {Cc, 1}));
      g.bytes = (static_cast<double>(R * Cc) + static_cast<double>(R)) * w;
    } else if (p.layout == 0) {  // contiguous
      g.out = view_of(OUT, o, {n}, {1});
      for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {n}, {1}));
      g.bytes = static_cast<double>(n) * w * (arity + 1);
    } else if (p.layout == 1) {  // strided: stride-2 of a 2x span, or a transposed 2-D view
      if (p.sub == 0) {
        g.out = view_of(OUT, o, {n}, {1});
        for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {n}, {2}));
      } else {
        g.out = view_of(OUT, o, {R, Cc}, {Cc, 1});
        for (int k = 0; k < arity; ++k) g.in.push_back(view_of(IN, off(rng), {R, Cc}, {1, R}));
      }
      g.bytes = static_cast<double>(n) * w * (arity + 1);
    } else {  // broadcast: a (1, C) row against (R, C), or a rank-0 scalar
      g.out = view_of(OUT, o, {R, Cc}, {Cc, 1});
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
  for (size_t pi = 0; pi < plans.size(); ++pi) {
    Gen& g = m.calls[pi];
    g.survives = tot[g.dt] - start[pi] <= cap[g.dt];
    m.survivors += g.survives;
  }
  return m;
}

// Poison every output arena (0xff bytes: NaN for the float dtypes) so a
// verified step can only pass on outputs it wrote itself.
void poison_outputs(Runtime& rt, const Mixed& m) {
  for (int d = 0; d < 4; ++d) rt.pool().fill(m.outA[d].buffer, 0xff);
}

// Recompute every surviving task of the stream with the oracle from the host
// copies of the inputs and compare with the GPU outputs (downloaded window by
// window): bit-exact, except float sums (<= 1 ulp, bit-exact share reported).
gbcheck::Tally verify_mixed(Runtime& rt, const Mixed& m) {
  gbcheck::Tally all;
  const gbcheck::Oracle& O = gbcheck::oracle();
  if (!O.ok) return all;
  const int orc_dt[4] = {ORC_F32, ORC_F16, ORC_BF16, ORC_I32};
  const int64_t kWindow = int64_t{64} << 20;  // elements per download window
  for (int d = 0; d < 4; ++d) {
    std::vector<uint32_t> idx;
    for (uint32_t i = 0; i < m.calls.size(); ++i)
      if (m.calls[i].dt == d && m.calls[i].survives) idx.push_back(i);
    std::sort(idx.begin(), idx.end(), [&](uint32_t a, uint32_t b) { return m.calls[a].out.offset < m.calls[b].out.offset; });
    const size_t w = gbcheck::width(orc_dt[d]);
    std::vector<unsigned char> win;
    size_t at = 0;
    while (at < idx.size()) {
      const int64_t wlo = m.calls[idx[at]].out.offset;
      size_t end = at;
      int64_t whi = wlo;
      while (end < idx.size()) {
        const Gen& g = m.calls[idx[end]];
        const int64_t e = g.out.offset + g.out.numel();
        if (e - wlo > kWindow && end > at) break;
        whi = std::max(whi, e);
        ++end;
      }
      win.resize(static_cast<size_t>(whi - wlo) * w);
      rt.pool().download_range(m.outA[d].buffer, static_cast<size_t>(wlo) * w, win.data(), win.size());
      gbcheck::Tally t = gbcheck::parallel_for(end - at, [&](size_t j, gbcheck::Tally& tl) {
        thread_local std::vector<unsigned char> scratch;
        const Gen& g = m.calls[idx[at + j]];
        const int64_t n = g.out.numel();
        scratch.assign(static_cast<size_t>(std::max<int64_t>(n, 1)) * w, 0);
        orc_view out = gbcheck::view(scratch.data(), orc_dt[d], 0, g.out.shape.data(), g.out.strides.data(),
                                     static_cast<int>(g.out.rank()));
        orc_view ins[2];
        for (int k = 0; k < g.in.n; ++k)
          ins[k] = gbcheck::view(const_cast<unsigned char*>(m.host_in[g.arena].data()), orc_dt[d], g.in.v[k].offset,
                                 g.in.v[k].shape.data(), g.in.v[k].strides.data(), static_cast<int>(g.in.v[k].rank()));
        int rc;
        if (g.op == OpKind::ReduceSum) rc = O.reduce(0, &out, ins);
        else rc = O.elementwise(static_cast<int>(g.op), &out, ins, g.in.n);
        if (rc != 0) {
          ++tl.tasks;
          ++tl.bad_tasks;
          if (tl.first.empty()) tl.first = "oracle error " + std::to_string(rc);
          return;
        }
        const bool float_sum = g.op == OpKind::ReduceSum && d != 3;
        gbcheck::compare(orc_dt[d], win.data() + static_cast<size_t>(g.out.offset - wlo) * w, scratch.data(), n,
                         float_sum ? gbcheck::kUlp1 : gbcheck::kExact, 0.0, tl, nullptr, "config2 task");
      });
      all.merge(t);
      at = end;
    }
  }
  return all;
}

void put_tally(const gbcheck::Tally& t, double* out) {  // mismatched tasks, checked tasks, elems, sum bit-exact frac, bad elems
  out[0] = gbcheck::oracle().ok ? static_cast<double>(t.bad_tasks) : -1.0;
  out[1] = static_cast<double>(t.tasks);
  out[2] = static_cast<double>(t.elems);
  out[3] = t.sum_elems ? static_cast<double>(t.sum_bitexact) / static_cast<double>(t.sum_elems) : 1.0;
  out[4] = static_cast<double>(t.bad_elems);
  if (!t.first.empty()) std::fprintf(stderr, "parity: first mismatch: %s\n", t.first.c_str());
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

// Load the parity checker (oracle/liboracle.so, path from bench.py).
int gb_set_oracle(const char* path) { return gbcheck::load_oracle(path) ? 0 : 1; }

// out: [0] tasks/s (device), [1] algorithmic GB/s, [2] tasks per step,
//      [3] mean bytes/task, [4] failed tasks, [5] host submit ns/task,
//      [6..10] parity of the last timed step (outputs poisoned before it):
//      mismatched tasks (-1 = no checker), checked tasks, checked elements,
//      bit-exact share of float-sum elements, mismatched elements
int gb_config2(int device, int n_tasks, int steps, double* out) {
  // GB_C2_FINITE=1 (diagnostics): device capacity -- the whole stream is
  // published with the workers stopped, then one finite generation drains it
  const bool finite = std::getenv("GB_C2_FINITE") != nullptr;
  Runtime rt(bench_cfg(device, finite ? static_cast<size_t>(n_tasks) + 2 : 4096));
  Mixed m = make_mixed(rt, n_tasks, 42);
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  Events ev(rt.device());
  std::vector<TaskHandle> hs;
  hs.reserve(m.calls.size());
  double dev_ms = 0, sub_ms = 0;
  uint64_t failed = 0;
  for (int s = 0; s < steps + 1; ++s) {  // step 0 warms up
    if (s == steps) poison_outputs(rt, m);  // outside the timed region
    hs.clear();
    double t_sub = 0;
    if (finite) {
      const double t0 = now_ms();
      for (const Gen& g : m.calls)
        hs.push_back(rt.submit_span(static_cast<uint64_t>(g.op), g.inputs(), g.out, std::span<const double>()));
      t_sub = now_ms() - t0;
      float kms = 0;
      check_abi(gpuos_dev_run_finite(rt.device(), &kms), "run_finite");
      rt.wait_all();
      if (s == 0) continue;
      dev_ms += kms;
      sub_ms += t_sub;
      for (const TaskHandle& h : hs) failed += h.state() == TaskState::Failed ? 1 : 0;
      continue;
    }
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
  hs.clear();
  const gbcheck::Tally t = verify_mixed(rt, m);
  const double tasks = static_cast<double>(m.calls.size()) * steps;
  out[0] = tasks / (dev_ms / 1e3);
  out[1] = m.bytes * steps / (dev_ms / 1e3) / 1e9;
  out[2] = static_cast<double>(m.calls.size());
  out[3] = m.bytes / static_cast<double>(m.calls.size());
  out[4] = static_cast<double>(failed);
  out[5] = sub_ms * 1e6 / tasks;
  put_tally(t, out + 6);
  return 0;
}

// out: [0] step us (median), [1] tasks/s, [2] GFLOP/s, [3] failed tasks,
//      [4] max relative error over the checked outputs,
//      [5..8] median us of the scale / QK^T / softmax / PV phases,
//      [9..13] parity (put_tally) of the last step: all heads, all phases
static int config3_impl(int device, int dtype, int steps, bool fenced, double* out) {
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
    if (s == steps + 1)  // the verified (last) step can only pass on its own outputs
      for (const TensorView* t : {&Qs, &Sc, &P, &O}) rt.pool().fill(t->buffer, 0xff);
    const double t0 = now_ms();
    if (fenced) hs.clear();
    for (int phase = 0; phase < 4; ++phase) {
      const double tp = now_ms();
      // device-dependency variant: the phases are ordered on the device by a
      // fence (Runtime::fence), one host wait per step instead of four
      if (fenced && phase > 0) rt.fence();
      if (!fenced) hs.clear();
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
      if (fenced) continue;
      for (const TaskHandle& th : hs) {
        th.wait();
        if (s >= 2) failed += th.state() == TaskState::Failed ? 1 : 0;
      }
      if (s >= 2) phase_us[phase].push_back((now_ms() - tp) * 1e3);
    }
    if (fenced) {
      rt.wait_all();
      for (const TaskHandle& th : hs)
        if (s >= 2) failed += th.state() == TaskState::Failed ? 1 : 0;
      for (int phase = 0; phase < 4; ++phase)
        if (s >= 2) phase_us[phase].push_back(0.0);
    }
    if (s >= 2) step_us.push_back((now_ms() - t0) * 1e3);
  }
  std::sort(step_us.begin(), step_us.end());
  const double med = step_us[step_us.size() / 2];
  // Parity of the last step (its outputs were poisoned before it), every
  // head and every phase, against the oracle applied to the GPU's own inputs
  // of that phase: scale exact; f32 matmul exact (fp64 ascending-k, as the
  // reference); bf16 matmul within the tensor-core bound; softmax rel 1e-6
  // (f32) / 1 ulp (bf16).
  gbcheck::Tally tally;
  if (gbcheck::oracle().ok) {
    const gbcheck::Oracle& Or = gbcheck::oracle();
    const int odt = dt == DType::F32 ? ORC_F32 : ORC_BF16;
    const size_t w = dtype_width(dt);
    auto fetch = [&](const TensorView& t, size_t n) {
      std::vector<unsigned char> b(n * w);
      rt.pool().download(t.buffer, b.data(), b.size());
      return b;
    };
    const size_t nqd = static_cast<size_t>(H) * S * D, nss = static_cast<size_t>(H) * S * S;
    auto hq = fetch(Q, nqd), hk = fetch(K, nqd), hv = fetch(V, nqd), hqs = fetch(Qs, nqd), hsc = fetch(Sc, nss),
         hp = fetch(P, nss), ho = fetch(O, nqd), hscale = fetch(scale, 1);
    std::vector<unsigned char> want(std::max(nqd, nss) / H * w);
    std::vector<double> bound(static_cast<size_t>(S) * S);
    auto vw = [&](std::vector<unsigned char>& b, int64_t off, int64_t r, int64_t c, int64_t s0, int64_t s1) {
      return gbcheck::view(b.data(), odt, off, {r, c}, {s0, s1});
    };
    // |A| @ |B| * k 2^-23 for the tensor-core bound (bf16 only)
    auto gemm_bound = [&](const std::vector<unsigned char>& A, int64_t ao, const std::vector<unsigned char>& B,
                          int64_t bo, int64_t M, int64_t K, int64_t N, int64_t bs0, int64_t bs1) {
      for (int64_t i = 0; i < M; ++i)
        for (int64_t j = 0; j < N; ++j) {
          double acc = 0;
          for (int64_t k = 0; k < K; ++k)
            acc += std::fabs(gbcheck::decode(odt, A.data(), ao + i * K + k)) *
                   std::fabs(gbcheck::decode(odt, B.data(), bo + k * bs0 + j * bs1));
          bound[static_cast<size_t>(i * N + j)] = static_cast<double>(K) * std::ldexp(1.0, -23) * acc;
        }
    };
    for (int h = 0; h < H; ++h) {
      const int64_t oq = static_cast<int64_t>(h) * S * D, os = static_cast<int64_t>(h) * S * S;
      // phase 0: Q * scale (rank-0 broadcast)
      orc_view o0 = gbcheck::view(want.data(), odt, 0, {S, D}, {D, 1});
      orc_view in0[2] = {vw(hq, oq, S, D, D, 1), gbcheck::view(hscale.data(), odt, 0, {}, {})};
      Or.elementwise(1, &o0, in0, 2);
      gbcheck::compare(odt, hqs.data() + oq * w, want.data(), S * D, gbcheck::kExact, 0, tally, nullptr, "scale");
      // phase 1: Q' K^T with K^T a transposed view
      orc_view o1 = gbcheck::view(want.data(), odt, 0, {S, S}, {S, 1});
      orc_view a1 = vw(hqs, oq, S, D, D, 1), b1 = vw(hk, oq, D, S, 1, D);
      Or.matmul(&o1, &a1, &b1, 256);
      if (dt == DType::F32) {
        gbcheck::compare(odt, hsc.data() + os * w, want.data(), S * S, gbcheck::kExact, 0, tally, nullptr, "qk_t");
      } else {
        gemm_bound(hqs, oq, hk, oq, S, D, S, 1, D);
        gbcheck::compare(odt, hsc.data() + os * w, want.data(), S * S, gbcheck::kGemm32, 0, tally, bound.data(), "qk_t");
      }
      // phase 2: row softmax
      orc_view o2 = gbcheck::view(want.data(), odt, 0, {S, S}, {S, 1});
      orc_view a2 = vw(hsc, os, S, S, S, 1);
      Or.softmax(&o2, &a2);
      gbcheck::compare(odt, hp.data() + os * w, want.data(), S * S, dt == DType::F32 ? gbcheck::kRel : gbcheck::kUlp1,
                       1e-6, tally, nullptr, "softmax");
      // phase 3: P V
      orc_view o3 = gbcheck::view(want.data(), odt, 0, {S, D}, {D, 1});
      orc_view a3 = vw(hp, os, S, S, S, 1), b3 = vw(hv, oq, S, D, D, 1);
      Or.matmul(&o3, &a3, &b3, 256);
      if (dt == DType::F32) {
        gbcheck::compare(odt, ho.data() + oq * w, want.data(), S * D, gbcheck::kExact, 0, tally, nullptr, "pv");
      } else {
        gemm_bound(hp, os, hv, oq, S, S, D, D, 1);
        gbcheck::compare(odt, ho.data() + oq * w, want.data(), S * D, gbcheck::kGemm32, 0, tally, bound.data(), "pv");
      }
    }
  }
  const double flops = 2.0 * H * (2.0 * S * S * D);  // QK^T + PV
  out[0] = med;
  out[1] = 4.0 * H / (med / 1e6);
  out[2] = flops / (med / 1e6) / 1e9;
  out[3] = static_cast<double>(failed);
  out[4] = tally.max_rel;
  for (int ph = 0; ph < 4; ++ph) {  // [5..8] median us of scale / QK^T / softmax / PV phases
    std::sort(phase_us[ph].begin(), phase_us[ph].end());
    out[5 + ph] = phase_us[ph][phase_us[ph].size() / 2];
  }
  put_tally(tally, out + 9);  // [9..13] parity of the last step, all 32 heads x 4 phases
  return 0;
}

// out: [0] tasks/s (device), [1] inject call ms (template compile + install),
//      [2] upload us, [3] epoch wait us, [4] bank write us, [5] flip us,
//      [6] checked rows, [7] rows not uniformly one variant, [8] rows with the
//      old variant after the swap window, [9] failed tasks, [10] canary hits,
//      [11] old rows, [12] new rows
int gb_config3(int device, int dtype, int steps, double* out) { return config3_impl(device, dtype, steps, false, out); }
// Device-dependency variant of config 3 (SURVEY §8(d) "report both"): the
// four phases are separated by Runtime::fence() instead of host waits.
int gb_config3_fenced(int device, int dtype, int steps, double* out) {
  return config3_impl(device, dtype, steps, true, out);
}

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

// Swap latency as SURVEY §8(d) config 4 defines it: inject_operator_at entry
// -> the first device dispatch of the id under the new table version (the
// device trace's dequeue stamp, converted to the host clock by the ping-pong
// calibration, +-1 us), with the ring busy: a stream of 4096-element tasks
// alternating builtin add and the injected op, re-injected `swaps` times.
// out: [0] p50 entry->first new dispatch us, [1] max, [2] p50 call-return ->
//      first new dispatch us, [3] p50 inject call us, [4] swaps measured,
//      [5] dispatches of the old version after the call returned (max over swaps),
//      [6] tasks/s of the traced stream
int gb_swap_latency(int device, int n_tasks, int swaps, double* out) {
  const int64_t E = 4096;
  RuntimeConfig cfg = bench_cfg(device, 4096);
  cfg.telemetry_enabled = true;
  cfg.trace_capacity = static_cast<size_t>(n_tasks) + 4096;
  Runtime rt(cfg);
  const double pa[2] = {1.5, -0.25}, pb[2] = {-2.0, 3.0};
  const uint32_t id = static_cast<uint32_t>(rt.inject_operator("scale_add", pa));
  TensorView IN = rt.alloc_tensor(DType::F32, {8 * E});
  TensorView OUT = rt.alloc_tensor(DType::F32, {1024 * E});
  rt.wait_all();
  struct Swap {
    uint64_t entry, exit, version;
  };
  std::vector<Swap> sw;
  const int every = n_tasks / (swaps + 1);
  const uint64_t t0 = monotonic_ns();
  for (int t = 0; t < n_tasks; ++t) {
    const TensorView in = view_of(IN, static_cast<int64_t>(t % 8) * E, {E}, {1});
    const TensorView o = view_of(OUT, static_cast<int64_t>(t % 1024) * E, {E}, {1});
    if (t % 2 == 0) rt.submit(OpKind::Add, {in, in}, o);
    else rt.submit(static_cast<uint64_t>(id), {in}, o);
    if (t > 0 && t % every == 0 && static_cast<int>(sw.size()) < swaps) {
      Swap s;
      s.entry = monotonic_ns();
      rt.inject_operator_at(id, "scale_add", (sw.size() % 2 == 0) ? std::span<const double>(pb, 2)
                                                                  : std::span<const double>(pa, 2));
      s.exit = monotonic_ns();
      s.version = rt.table().snapshot_version();
      sw.push_back(s);
    }
  }
  rt.wait_all();
  const double secs = static_cast<double>(monotonic_ns() - t0) / 1e9;
  const std::vector<Tracepoint> tr = rt.trace();
  std::vector<double> lat_entry, lat_exit, call;
  uint64_t late_old_max = 0;
  for (const Swap& s : sw) {
    uint64_t first = UINT64_MAX, late_old = 0;
    for (const Tracepoint& p : tr) {
      if (p.op_id != id) continue;
      if (p.version >= s.version && p.dequeue_ns >= s.entry && p.dequeue_ns < first) first = p.dequeue_ns;
      if (p.version < s.version && p.dequeue_ns > s.exit) ++late_old;
    }
    if (first == UINT64_MAX) continue;
    lat_entry.push_back(static_cast<double>(first - s.entry) / 1e3);
    lat_exit.push_back(static_cast<double>(static_cast<int64_t>(first - s.exit)) / 1e3);
    call.push_back(static_cast<double>(s.exit - s.entry) / 1e3);
    late_old_max = std::max(late_old_max, late_old);
  }
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? -1.0 : v[v.size() / 2];
  };
  out[0] = med(lat_entry);
  out[1] = lat_entry.empty() ? -1.0 : *std::max_element(lat_entry.begin(), lat_entry.end());
  out[2] = med(lat_exit);
  out[3] = med(call);
  out[4] = static_cast<double>(lat_entry.size());
  out[5] = static_cast<double>(late_old_max);
  out[6] = n_tasks / secs;
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

// Config 5: independent task streams of the config-2
// distribution (stream s has seed 42 + s), stream s on GPU s mod G.  This
// process owns one GPU and the streams `ids` assigned to it; each stream has
// its own host producer thread and its own runtime (ring + persistent
// generation of `workers` CTAs: the streams on a GPU split its SMs).
// gb_c5_open builds the streams (outside any timed region), gb_c5_run times
// them concurrently: the producers start together at a host barrier, and the
// device time is the union of the streams' worker-kernel lifetimes (earliest
// start event to latest exit event, all on this device) -- bench.py takes
// the max of that over ranks after a barrier.
struct C5Stream {
  std::unique_ptr<Runtime> rt;
  Mixed m;
  void *e0 = nullptr, *e1 = nullptr, *ks = nullptr;
  double submit_ms = 0;
  uint64_t failed = 0;
};
struct C5 {
  std::vector<std::unique_ptr<C5Stream>> ss;
};

void* gb_c5_open(int device, const int* ids, int n, int tasks_per_stream, int workers, long long out_cap) {
  auto* c = new C5();
  c->ss.resize(static_cast<size_t>(n));
  std::vector<std::thread> th;
  for (int i = 0; i < n; ++i) {
    c->ss[static_cast<size_t>(i)] = std::make_unique<C5Stream>();
    C5Stream* st = c->ss[static_cast<size_t>(i)].get();
    RuntimeConfig cfg = bench_cfg(device, 4096);
    cfg.workers.num_workers = static_cast<size_t>(workers);
    st->rt = std::make_unique<Runtime>(cfg);
    const uint64_t seed = 42 + static_cast<uint64_t>(ids[i]);
    th.emplace_back([st, tasks_per_stream, seed, out_cap] {
      st->m = make_mixed(*st->rt, tasks_per_stream, seed, out_cap);
    });
  }
  for (auto& t : th) t.join();
  for (auto& st : c->ss) {
    st->rt->wait_all();
    check_abi(gpuos_event_create(st->rt->device(), &st->e0), "ev");
    check_abi(gpuos_event_create(st->rt->device(), &st->e1), "ev");
    check_abi(gpuos_dev_kernel_stream(st->rt->device(), &st->ks), "ks");
    check_abi(gpuos_dev_stop(st->rt->device()), "stop");
  }
  return c;
}

// One generation of stream `st`: start (events bracket the kernel), submit
// the whole stream, drain, stop.
static void c5_stream(C5Stream& st, std::atomic<int>* gate, int n_streams) {
  Runtime& rt = *st.rt;
  std::vector<TaskHandle> hs;
  hs.reserve(st.m.calls.size());
  if (gate) {  // all producers start together
    gate->fetch_add(1);
    while (gate->load() < n_streams) _mm_pause();
  }
  check_abi(gpuos_event_record(rt.device(), st.e0, st.ks), "ev0");
  check_abi(gpuos_dev_start(rt.device()), "start");
  check_abi(gpuos_event_record(rt.device(), st.e1, st.ks), "ev1");
  const double t0 = now_ms();
  for (const Gen& g : st.m.calls)
    hs.push_back(rt.submit_span(static_cast<uint64_t>(g.op), g.inputs(), g.out, std::span<const double>()));
  st.submit_ms = now_ms() - t0;
  rt.wait_all();
  check_abi(gpuos_dev_stop(rt.device()), "stop");
  check_abi(gpuos_event_sync(rt.device(), st.e1), "sync");
  st.failed = 0;
  for (const TaskHandle& h : hs) st.failed += h.state() == TaskState::Failed ? 1 : 0;
}

// out: [0] tasks run, [1] union device ms, [2] algorithmic bytes, [3] failed,
//      [4..8] parity (put_tally, -1 when verify == 0), [9] host submit ns/task
//      (mean over streams), [10] slowest single stream ms
int gb_c5_run(void* h, int warm, int verify, double* out) {
  auto* c = static_cast<C5*>(h);
  const int n = static_cast<int>(c->ss.size());
  if (warm)
    for (auto& st : c->ss) c5_stream(*st, nullptr, 1);  // each stream alone
  if (verify)
    for (auto& st : c->ss) poison_outputs(*st->rt, st->m);
  std::atomic<int> gate{0};
  std::vector<std::thread> th;
  for (auto& st : c->ss) th.emplace_back([&, p = st.get()] { c5_stream(*p, &gate, n); });
  for (auto& t : th) t.join();
  // union of the kernel lifetimes, relative to stream 0's start event
  double lo = 0, hi = 0, slow = 0, bytes = 0, sub = 0;
  uint64_t tasks = 0, failed = 0;
  for (auto& st : c->ss) {
    float a = 0, b = 0, own = 0;
    check_abi(gpuos_event_elapsed_ms(st->rt->device(), c->ss[0]->e0, st->e0, &a), "elapsed");
    check_abi(gpuos_event_elapsed_ms(st->rt->device(), c->ss[0]->e0, st->e1, &b), "elapsed");
    check_abi(gpuos_event_elapsed_ms(st->rt->device(), st->e0, st->e1, &own), "elapsed");
    lo = std::min(lo, static_cast<double>(a));
    hi = std::max(hi, static_cast<double>(b));
    slow = std::max(slow, static_cast<double>(own));
    bytes += st->m.bytes;
    tasks += st->m.calls.size();
    failed += st->failed;
    sub += st->submit_ms * 1e6 / static_cast<double>(st->m.calls.size());
  }
  gbcheck::Tally t;
  if (verify)
    for (auto& st : c->ss) t.merge(verify_mixed(*st->rt, st->m));
  out[0] = static_cast<double>(tasks);
  out[1] = hi - lo;
  out[2] = bytes;
  out[3] = static_cast<double>(failed);
  if (verify) {
    put_tally(t, out + 4);
  } else {
    for (int i = 4; i < 9; ++i) out[i] = -1;
  }
  out[9] = sub / n;
  out[10] = slow;
  return 0;
}

// Tasks whose outputs survive the output-ring wrap (the checkable ones).
double gb_c5_survivors(void* h) {
  double s = 0;
  for (auto& st : static_cast<C5*>(h)->ss) s += static_cast<double>(st->m.survivors);
  return s;
}

void gb_c5_close(void* h) {
  auto* c = static_cast<C5*>(h);
  for (auto& st : c->ss) {
    gpuos_event_destroy(st->rt->device(), st->e0);
    gpuos_event_destroy(st->rt->device(), st->e1);
    gpuos_dev_start(st->rt->device());  // the runtime's shutdown drains a resident generation
  }
  delete c;
}

}  // extern "C"
