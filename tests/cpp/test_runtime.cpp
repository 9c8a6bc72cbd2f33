// Runtime parity suite on the B200 (restates reference tests/test_runtime.cpp,
// test_executor.cpp and acceptance criteria C2/C3/C7 against gpuos::Runtime):
// lifecycle, routing, overflow fallback, injection and kill, error codes,
// queue-vs-inline equivalence, accounting identities, hot-swap under load,
// drain-on-shutdown.  Built by `make cpp-tests`, run by tests/test_cpp_gpu.py.
#include <gpuos/runtime.hpp>

#include <unistd.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <random>
#include <sstream>
#include <thread>
#include <vector>

#include "check.hpp"
#include "../../tools/bench/oracle_check.hpp"

using namespace gpuos;

namespace {

bool close_tol(double got, double want, double tol) {
  if (std::isnan(got) || std::isnan(want)) return std::isnan(got) && std::isnan(want);
  return std::abs(got - want) <= tol * std::max(1.0, std::abs(want));
}

std::vector<double> read_all(Runtime& rt, const TensorView& v) {
  BoundView b(rt.pool(), v);
  std::vector<double> out(static_cast<size_t>(v.numel()));
  for (size_t i = 0; i < out.size(); ++i) out[i] = b.load(static_cast<int64_t>(i));
  return out;
}

void fill(Runtime& rt, const TensorView& v, const std::vector<double>& vals) {
  BoundView b(rt.pool(), v);
  for (size_t i = 0; i < vals.size(); ++i) b.store(static_cast<int64_t>(i), vals[i]);
}

std::vector<double> random_vals(std::mt19937_64& rng, size_t n, double lo = -4.0, double hi = 4.0) {
  std::uniform_real_distribution<double> d(lo, hi);
  std::vector<double> v(n);
  for (double& x : v) x = d(rng);
  return v;
}

RuntimeConfig small_config(size_t capacity = 256, size_t workers = 8) {
  RuntimeConfig c;
  c.capacity = capacity;
  c.workers.num_workers = workers;
  return c;
}

double f32(double x) { return static_cast<double>(static_cast<float>(x)); }

}  // namespace

TEST_CASE("config from env") {
  ::setenv("GPUOS_CAPACITY", "128", 1);
  ::setenv("GPUOS_WORKERS", "3", 1);
  ::setenv("GPUOS_YIELD_EVERY", "5", 1);
  ::setenv("GPUOS_MAX_ELEMS", "1000", 1);
  RuntimeConfig env = RuntimeConfig::from_env();
  CHECK(env.capacity == 128);
  CHECK(env.workers.num_workers == 3);
  CHECK(env.workers.yield_every == 5);
  CHECK(env.max_elements == 1000);
  ::setenv("GPUOS_CAPACITY", "not-a-number", 1);
  ::setenv("GPUOS_WORKERS", "", 1);
  ::setenv("GPUOS_MAX_ELEMS", "12x", 1);
  env = RuntimeConfig::from_env();
  CHECK(env.capacity == 4096);
  CHECK(env.workers.num_workers == 0);
  CHECK(env.max_elements == 65536);
  ::unsetenv("GPUOS_CAPACITY");
  ::unsetenv("GPUOS_WORKERS");
  ::unsetenv("GPUOS_YIELD_EVERY");
  ::unsetenv("GPUOS_MAX_ELEMS");
  const RuntimeConfig d;
  CHECK(d.capacity == 4096);
  CHECK(d.max_elements == 65536);
  CHECK(d.max_chain == 8);
  CHECK(d.max_sdpa_context == 2048);
  CHECK_FALSE(d.fusion_enabled);
}

TEST_CASE("runtime starts with the builtin set at version 15") {
  Runtime rt(small_config(256, 2));
  REQUIRE(rt.worker_alive());
  REQUIRE(rt.num_workers() == 2);
  REQUIRE_FALSE(rt.stopped());
  REQUIRE(rt.table().snapshot_version() == kNumBuiltinOps + 1);
  REQUIRE(rt.table().latest_entry(static_cast<uint64_t>(OpKind::Relu)).status == OpStatus::Active);
  REQUIRE(rt.table().latest_entry(kCompositeOpId).status == OpStatus::Active);
  REQUIRE(rt.table().latest_entry(40).status == OpStatus::Empty);
  const TaskQueue::Snapshot s = rt.peek_queue();
  REQUIRE(s.head == 0);
  REQUIRE(s.tail == 0);
  REQUIRE(s.processed == 0);
}

TEST_CASE("init, shutdown, init again leaves no residue") {
  for (int round = 0; round < 2; ++round) {
    Runtime rt(small_config(16, 2));
    REQUIRE(rt.worker_alive());
    auto a = rt.alloc_tensor(DType::F32, {32});
    auto out = rt.alloc_tensor(DType::F32, {32});
    fill(rt, a, std::vector<double>(32, 2.0));
    auto h = rt.submit(OpKind::Relu, {a}, out);
    REQUIRE(rt.wait(h) == TaskState::Done);
    rt.shutdown();
    REQUIRE_FALSE(rt.worker_alive());
    REQUIRE(rt.stopped());
    rt.shutdown();
    auto late = rt.submit(OpKind::Relu, {a}, out);
    REQUIRE(late.state() == TaskState::Failed);
    REQUIRE(late.error() == ErrorCode::RuntimeStopped);
  }
}

TEST_CASE("small elementwise work routes to the persistent workers, bit-exact") {
  Runtime rt(small_config());
  std::mt19937_64 rng(101);
  auto a = rt.alloc_tensor(DType::F32, {1024});
  auto b = rt.alloc_tensor(DType::F32, {1024});
  auto out = rt.alloc_tensor(DType::F32, {1024});
  const auto va = random_vals(rng, 1024), vb = random_vals(rng, 1024);
  fill(rt, a, va);
  fill(rt, b, vb);
  auto h = rt.submit(OpKind::Add, {a, b}, out);
  REQUIRE(rt.wait(h) == TaskState::Done);
  const CounterSnapshot c = rt.counters();
  CHECK(c.submitted == 1);
  CHECK(c.committed == 1);
  CHECK(c.inline_executions == 0);
  CHECK(c.processed == 1);
  const auto got = read_all(rt, out);
  for (size_t i = 0; i < got.size(); ++i) REQUIRE(got[i] == f32(f32(va[i]) + f32(vb[i])));
}

TEST_CASE("large matmul executes inline on the conventional path") {
  Runtime rt(small_config());
  std::mt19937_64 rng(202);
  const int64_t n = 512;
  auto a = rt.alloc_tensor(DType::F32, {n, n});
  auto b = rt.alloc_tensor(DType::F32, {n, n});
  auto out = rt.alloc_tensor(DType::F32, {n, n});
  const auto va = random_vals(rng, static_cast<size_t>(n * n), -1.0, 1.0);
  const auto vb = random_vals(rng, static_cast<size_t>(n * n), -1.0, 1.0);
  fill(rt, a, va);
  fill(rt, b, vb);
  auto h = rt.submit(OpKind::MatMulSmall, {a, b}, out);
  REQUIRE(h.state() == TaskState::Done);  // inline is synchronous
  const CounterSnapshot c = rt.counters();
  CHECK(c.inline_executions == 1);
  CHECK(c.committed == 0);
  BoundView bo(rt.pool(), out);
  std::uniform_int_distribution<int64_t> pick(0, n - 1);
  for (int t = 0; t < 12; ++t) {
    const int64_t i = pick(rng), j = pick(rng);
    double want = 0.0;
    for (int64_t k = 0; k < n; ++k) want += f32(va[static_cast<size_t>(i * n + k)]) * f32(vb[static_cast<size_t>(k * n + j)]);
    REQUIRE(close_tol(bo.load(i * n + j), want, 1e-6));
  }
}

TEST_CASE("small matmul is queued and bit-exact against double ascending-k") {
  Runtime rt(small_config());
  std::mt19937_64 rng(203);
  const int64_t m = 128, k = 64, n = 128;
  auto a = rt.alloc_tensor(DType::F32, {m, k});
  auto kt = rt.alloc_tensor(DType::F32, {n, k});  // K, used transposed
  auto out = rt.alloc_tensor(DType::F32, {m, n});
  const auto va = random_vals(rng, static_cast<size_t>(m * k), -1.0, 1.0);
  const auto vk = random_vals(rng, static_cast<size_t>(n * k), -1.0, 1.0);
  fill(rt, a, va);
  fill(rt, kt, vk);
  TensorView kview = kt;  // (k, n) view of K with strides swapped
  kview.shape = {k, n};
  kview.strides = {1, k};
  REQUIRE(rt.wait(rt.submit(OpKind::MatMulSmall, {a, kview}, out)) == TaskState::Done);
  CHECK(rt.counters().committed == 1);
  const auto got = read_all(rt, out);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) acc += f32(va[static_cast<size_t>(i * k + p)]) * f32(vk[static_cast<size_t>(j * k + p)]);
      REQUIRE(got[static_cast<size_t>(i * n + j)] == f32(acc));
    }
}

TEST_CASE("work ceiling splits routing at the element boundary") {
  RuntimeConfig cfg = small_config();
  cfg.max_elements = 4096;
  Runtime rt(cfg);
  auto si = rt.alloc_tensor(DType::F32, {4096});
  auto so = rt.alloc_tensor(DType::F32, {4096});
  auto bi = rt.alloc_tensor(DType::F32, {4097});
  auto bo = rt.alloc_tensor(DType::F32, {4097});
  fill(rt, si, std::vector<double>(4096, -1.5));
  fill(rt, bi, std::vector<double>(4097, -1.5));
  rt.wait(rt.submit(OpKind::Relu, {si}, so));
  CounterSnapshot c = rt.counters();
  CHECK(c.committed == 1);
  CHECK(c.inline_executions == 0);
  rt.wait(rt.submit(OpKind::Relu, {bi}, bo));
  c = rt.counters();
  CHECK(c.committed == 1);
  CHECK(c.inline_executions == 1);
  CHECK(read_all(rt, so) == std::vector<double>(4096, 0.0));
  CHECK(read_all(rt, bo) == std::vector<double>(4097, 0.0));
}

TEST_CASE("attention context bound gates queue routing") {
  RuntimeConfig cfg = small_config();
  cfg.max_elements = 1u << 20;
  Runtime rt(cfg);
  std::mt19937_64 rng(303);
  const int64_t h = 1, d = 8;
  for (const int64_t t : {int64_t{2048}, int64_t{2049}}) {
    auto q = rt.alloc_tensor(DType::F32, {h, d});
    auto k = rt.alloc_tensor(DType::F32, {h, t, d});
    auto v = rt.alloc_tensor(DType::F32, {h, t, d});
    auto out = rt.alloc_tensor(DType::F32, {h, d});
    fill(rt, q, random_vals(rng, static_cast<size_t>(h * d)));
    fill(rt, k, random_vals(rng, static_cast<size_t>(h * t * d), -1.0, 1.0));
    fill(rt, v, random_vals(rng, static_cast<size_t>(h * t * d), -1.0, 1.0));
    const CounterSnapshot before = rt.counters();
    REQUIRE(rt.wait(rt.submit(OpKind::Sdpa, {q, k, v}, out)) == TaskState::Done);
    const CounterSnapshot after = rt.counters();
    if (t <= 2048) CHECK(after.committed == before.committed + 1);
    else CHECK(after.inline_executions == before.inline_executions + 1);
  }
}

TEST_CASE("queue overflow falls back to inline execution without loss") {
  Runtime rt(small_config(4, 1));
  // hold the workers so the 4-slot ring fills (the reference pins its single
  // worker with a gated host lambda, test_runtime.cpp:243-256)
  check_abi(gpuos_dev_hold(rt.device(), 1), "hold");
  constexpr int kTasks = 32;
  std::vector<TensorView> outs;
  std::vector<TaskHandle> hs;
  for (int t = 0; t < kTasks; ++t) {
    auto a = rt.alloc_tensor(DType::F32, {8});
    auto b = rt.alloc_tensor(DType::F32, {8});
    auto out = rt.alloc_tensor(DType::F32, {8});
    fill(rt, a, std::vector<double>(8, t));
    fill(rt, b, std::vector<double>(8, 100.0));
    outs.push_back(out);
    hs.push_back(rt.submit(OpKind::Add, {a, b}, out));
  }
  const CounterSnapshot mid = rt.counters();
  REQUIRE(mid.queue_full_fallbacks > 0);
  REQUIRE(mid.submitted == kTasks);
  REQUIRE(mid.committed + mid.inline_executions == mid.submitted);
  check_abi(gpuos_dev_hold(rt.device(), 0), "release");
  rt.wait_all();
  for (int t = 0; t < kTasks; ++t) {
    REQUIRE(hs[static_cast<size_t>(t)].state() == TaskState::Done);
    REQUIRE(read_all(rt, outs[static_cast<size_t>(t)]) == std::vector<double>(8, 100.0 + t));
  }
  const CounterSnapshot done = rt.counters();
  CHECK(done.processed == done.committed);
  CHECK(done.failed == 0);
}

TEST_CASE("injected operators: ids, exact values, cache, audit") {
  Runtime rt(small_config());
  const double p[2] = {2.0, -1.0};
  const uint64_t id = rt.inject_operator("scale_add", p);
  REQUIRE(id == kFirstInjectedId);
  auto x = rt.alloc_tensor(DType::F32, {1});
  auto y = rt.alloc_tensor(DType::F32, {1});
  fill(rt, x, {1.5});
  REQUIRE(rt.wait(rt.submit(id, {x}, y)) == TaskState::Done);
  REQUIRE(read_all(rt, y)[0] == 2.0);
  CHECK(rt.counters().committed == 1);
  // same signature -> cache hit; different params -> new module and id
  const uint64_t id2 = rt.inject_operator("scale_add", p);
  CHECK(id2 == kFirstInjectedId + 1);
  CHECK(rt.module_cache().compiles() == 1);
  CHECK(rt.counters().cache_hits == 1);
  const double q[2] = {3.0, 0.5};
  const uint64_t id3 = rt.inject_operator("scale_add", q);
  auto y3 = rt.alloc_tensor(DType::F32, {1});
  REQUIRE(rt.wait(rt.submit(id3, {x}, y3)) == TaskState::Done);
  CHECK(read_all(rt, y3)[0] == 5.0);
  CHECK(rt.counters().injections == 3);
  const auto audit = rt.table().audit();
  REQUIRE(!audit.empty());
  CHECK(audit.back().template_name == "scale_add");
  CHECK(audit.back().version == rt.table().snapshot_version());
  std::stringstream ss;
  rt.table().export_audit_jsonl(ss);
  const auto parsed = OperatorTable::parse_audit_jsonl(ss);
  REQUIRE(parsed.size() == audit.size());
  for (size_t i = 0; i < parsed.size(); ++i) {
    CHECK(parsed[i].op_id == audit[i].op_id);
    CHECK(parsed[i].signature == audit[i].signature);
    CHECK(parsed[i].params == audit[i].params);
    CHECK(parsed[i].version == audit[i].version);
    CHECK(parsed[i].ts_ns == audit[i].ts_ns);
  }
  for (size_t i = 1; i < parsed.size(); ++i) CHECK(parsed[i].ts_ns > parsed[i - 1].ts_ns);
}

TEST_CASE("injected relu matches the builtin bit for bit, every template exact") {
  Runtime rt(small_config());
  rt.templates().add({"my_relu", "max(in0, 0)", 1});
  const uint64_t id = rt.inject_operator("my_relu");
  std::mt19937_64 rng(505);
  const auto vals = random_vals(rng, 4096);
  auto x = rt.alloc_tensor(DType::F32, {4096});
  auto y1 = rt.alloc_tensor(DType::F32, {4096});
  auto y2 = rt.alloc_tensor(DType::F32, {4096});
  fill(rt, x, vals);
  REQUIRE(rt.wait(rt.submit(OpKind::Relu, {x}, y1)) == TaskState::Done);
  REQUIRE(rt.wait(rt.submit(id, {x}, y2)) == TaskState::Done);
  REQUIRE(read_all(rt, y1) == read_all(rt, y2));
  // every shipped template vs narrow_to(eval_expr) (test_opcompiler.cpp:528-558)
  for (const std::string& name : rt.templates().names()) {
    const OperatorTemplate t = rt.templates().get(name);
    const double params[8] = {0.75, 2.5, 0, 0, 0, 0, 0, 0};
    const uint64_t oid = rt.inject_operator(name, params);
    std::vector<TensorView> ins;
    std::vector<std::vector<double>> iv;
    for (int i = 0; i < t.arity; ++i) {
      ins.push_back(rt.alloc_tensor(DType::F64, {257}));
      iv.push_back(random_vals(rng, 257, -3.0, 3.0));
      fill(rt, ins.back(), iv.back());
    }
    auto out = rt.alloc_tensor(DType::F64, {257});
    // module dtype F32 vs F64 output -> DTypeMismatch, then a F64 module
    auto hm = rt.submit(oid, ins, out);
    REQUIRE(rt.wait(hm) == TaskState::Failed);
    CHECK(hm.error() == ErrorCode::DTypeMismatch);
    const uint64_t oid64 = rt.inject_operator(name, params, DType::F64);
    REQUIRE(rt.wait(rt.submit(oid64, ins, out)) == TaskState::Done);
    const ExprPtr ast = parse_expression(t.source);
    const auto got = read_all(rt, out);
    for (size_t e = 0; e < 257; ++e) {
      double in[4] = {0, 0, 0, 0};
      for (int i = 0; i < t.arity; ++i) in[i] = iv[static_cast<size_t>(i)][e];
      const double want = eval_expr(*ast, {in, 4}, {params, 8});
      // + - * / sqrt abs max min are exact; exp/tanh allow 2 ulp of libdevice vs glibc
      if (name == "sigmoid" || name == "silu" || name == "tanh_gate")
        REQUIRE(close_tol(got[e], want, 4e-16));
      else
        REQUIRE((got[e] == want || (std::isnan(got[e]) && std::isnan(want))));
    }
  }
}

TEST_CASE("kill fails fast and re-injection revives the id") {
  Runtime rt(small_config());
  const double p[2] = {1.0, 0.0};
  const uint64_t id = rt.inject_operator("scale_add", p);
  auto x = rt.alloc_tensor(DType::F32, {16});
  auto y = rt.alloc_tensor(DType::F32, {16});
  REQUIRE(rt.wait(rt.submit(id, {x}, y)) == TaskState::Done);
  const uint64_t v0 = rt.table().snapshot_version();
  rt.kill_operator(static_cast<uint32_t>(id));
  CHECK(rt.table().snapshot_version() == v0 + 1);
  auto h = rt.submit(id, {x}, y);
  REQUIRE(rt.wait(h) == TaskState::Failed);
  REQUIRE(h.error() == ErrorCode::OperatorKilled);
  // a killed builtin stays eligible and fails on the worker
  rt.kill_operator(static_cast<uint32_t>(OpKind::Relu));
  const uint64_t committed = rt.counters().committed;
  auto h2 = rt.submit(OpKind::Relu, {x}, y);
  REQUIRE(rt.wait(h2) == TaskState::Failed);
  REQUIRE(h2.error() == ErrorCode::OperatorKilled);
  CHECK(rt.counters().committed == committed + 1);
  rt.inject_operator_at(static_cast<uint32_t>(id), "scale_add", p);
  REQUIRE(rt.wait(rt.submit(id, {x}, y)) == TaskState::Done);
  CHECK_THROWS_AS(rt.inject_operator_at(5, "scale_add", p), Error);
  CHECK_THROWS_AS(rt.inject_operator_at(5000, "scale_add", p), Error);
  CHECK_THROWS_AS(rt.inject_operator("no_such_template"), Error);
}

TEST_CASE("bad calls fail on the handle with the reference error codes") {
  Runtime rt(small_config());
  auto x = rt.alloc_tensor(DType::F32, {8});
  auto y = rt.alloc_tensor(DType::F32, {8});
  auto h1 = rt.submit(40, {x}, y);  // never injected: inline, NotInstalled
  REQUIRE(rt.wait(h1) == TaskState::Failed);
  REQUIRE(h1.error() == ErrorCode::NotInstalled);
  auto h2 = rt.submit(uint64_t{1} << 33, {x}, y);
  REQUIRE(rt.wait(h2) == TaskState::Failed);
  REQUIRE(h2.error() == ErrorCode::OutOfRange);
  TensorView bogus = x;
  bogus.buffer = 999999;
  auto h3 = rt.submit(OpKind::Relu, {bogus}, y);
  REQUIRE(rt.wait(h3) == TaskState::Failed);
  REQUIRE(h3.error() == ErrorCode::InvalidBuffer);
  auto h4 = rt.submit(OpKind::Add, {x}, y);
  REQUIRE(rt.wait(h4) == TaskState::Failed);
  REQUIRE(h4.error() == ErrorCode::ArityError);
  auto h5 = rt.submit(OpKind::Add, std::vector<TensorView>{x, x, x, x, x}, y);
  REQUIRE(h5.error() == ErrorCode::ArityError);
  auto xi = rt.alloc_tensor(DType::I32, {8});
  auto h6 = rt.submit(OpKind::Gelu, {xi}, xi);
  REQUIRE(rt.wait(h6) == TaskState::Failed);
  REQUIRE(h6.error() == ErrorCode::DTypeMismatch);
  auto e = rt.alloc_tensor(DType::F32, {3, 0});
  auto eo = rt.alloc_tensor(DType::F32, {3});
  auto h7 = rt.submit(OpKind::ReduceMax, {e}, eo);
  REQUIRE(rt.wait(h7) == TaskState::Failed);
  REQUIRE(h7.error() == ErrorCode::EmptyAxis);
  REQUIRE(rt.worker_alive());
  REQUIRE(rt.wait(rt.submit(OpKind::Relu, {x}, y)) == TaskState::Done);
  TaskHandle invalid;
  CHECK_FALSE(invalid.valid());
  CHECK_THROWS_AS(invalid.state(), Error);
}

TEST_CASE("queue and inline paths agree bit for bit") {
  RuntimeConfig qc = small_config();
  RuntimeConfig ic = small_config();
  ic.max_elements = 0;  // everything inline
  Runtime rq(qc), ri(ic);
  std::mt19937_64 rng(707);
  auto run_both = [&](OpKind k, const std::vector<std::vector<int64_t>>& in_shapes, const std::vector<int64_t>& out_shape,
                      std::vector<double> scalars, DType dt) {
    std::vector<std::vector<double>> vals;
    std::vector<TensorView> iq, ii;
    for (const auto& s : in_shapes) {
      iq.push_back(rq.alloc_tensor(dt, Shape(s)));
      ii.push_back(ri.alloc_tensor(dt, Shape(s)));
      vals.push_back(random_vals(rng, static_cast<size_t>(iq.back().numel()), -2.0, 2.0));
      fill(rq, iq.back(), vals.back());
      fill(ri, ii.back(), vals.back());
    }
    auto oq = rq.alloc_tensor(dt, Shape(out_shape));
    auto oi = ri.alloc_tensor(dt, Shape(out_shape));
    REQUIRE(rq.wait(rq.submit(static_cast<uint64_t>(k), iq, oq, scalars)) == TaskState::Done);
    REQUIRE(ri.wait(ri.submit(static_cast<uint64_t>(k), ii, oi, scalars)) == TaskState::Done);
    REQUIRE(read_all(rq, oq) == read_all(ri, oi));
  };
  run_both(OpKind::Add, {{64, 33}, {1, 33}}, {64, 33}, {}, DType::F32);
  run_both(OpKind::Gelu, {{1000}}, {1000}, {}, DType::F32);
  run_both(OpKind::Softmax, {{16, 128}}, {16, 128}, {}, DType::F32);
  run_both(OpKind::LayerNorm, {{8, 96}, {96}, {96}}, {8, 96}, {1e-5}, DType::F64);
  run_both(OpKind::ReduceSum, {{32, 1500}}, {32}, {}, DType::F32);
  run_both(OpKind::Rope, {{6, 64}, {6}}, {6, 64}, {}, DType::F64);
  run_both(OpKind::Sdpa, {{4, 64}, {4, 300, 64}, {4, 300, 64}}, {4, 64}, {}, DType::F32);
  run_both(OpKind::Mul, {{3000}, {3000}}, {3000}, {}, DType::BF16);
  CHECK(ri.counters().committed == 0);
}

TEST_CASE("accounting identity holds at quiescence") {
  Runtime rt(small_config(64, 4));
  auto x = rt.alloc_tensor(DType::F32, {4096});
  auto y = rt.alloc_tensor(DType::F32, {4096});
  auto big = rt.alloc_tensor(DType::F32, {70000});
  for (int i = 0; i < 500; ++i) {
    rt.submit(OpKind::Relu, {x}, y);
    if (i % 50 == 0) rt.submit(OpKind::Relu, {big}, big);
  }
  rt.submit(OpKind::Add, {x}, y);  // fails on the worker
  rt.wait_all();
  const CounterSnapshot c = rt.counters();
  CHECK(c.submitted == c.inline_executions + c.committed + rt.fusion_absorbed());
  CHECK(c.processed == c.committed);
  CHECK(c.failed == 1);
  const auto s = rt.peek_queue();
  CHECK(s.processed == s.head);
  CHECK(s.head == s.tail);
}

// Reference C1 (acceptance_main.cpp:80-212) and test_queue.cpp:292-361 on the
// device ring: a monitor thread samples peek_queue() continuously while one
// producer streams 10^5 tasks through compact (dense) and extended
// (broadcast scalar) slots; the cursor invariant processed <= head <= tail
// must hold in every sample and every cursor must be monotone.  Exactly-once:
// each task's output region is a function of its sequence number, every
// handle completes Done, and the device trace holds every sequence number
// exactly once (xor and count, as the reference checks).
TEST_CASE("live ring invariants: processed <= head <= tail under load, every task exactly once") {
  RuntimeConfig cfg = small_config(1024, 0);
  cfg.telemetry_enabled = true;
  const int n = 100000, len = 64;
  cfg.trace_capacity = n + 1024;
  Runtime rt(cfg);
  auto x = rt.alloc_tensor(DType::F32, {len});
  auto consts = rt.alloc_tensor(DType::F32, {n});
  auto out = rt.alloc_tensor(DType::F32, {int64_t{n} * len});
  std::vector<double> xv(len), cv(n);
  for (int i = 0; i < len; ++i) xv[i] = i * 0.5;
  for (int i = 0; i < n; ++i) cv[i] = static_cast<double>(i % 4096);
  fill(rt, x, xv);
  fill(rt, consts, cv);
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> samples{0}, violations{0}, regressions{0};
  std::thread monitor([&] {
    TaskQueue::Snapshot last{};
    while (!stop.load(std::memory_order_acquire)) {
      const TaskQueue::Snapshot s = rt.peek_queue();
      if (!(s.processed <= s.head && s.head <= s.tail)) violations.fetch_add(1);
      if (s.processed < last.processed || s.head < last.head || s.tail < last.tail) regressions.fetch_add(1);
      last = s;
      samples.fetch_add(1);
    }
  });
  std::vector<TaskHandle> hs;
  hs.reserve(n);
  for (int i = 0; i < n; ++i) {
    TensorView o = out;
    o.shape = {len};
    o.strides = {1};
    o.offset = int64_t{i} * len;
    if (i % 2 == 0) {
      // compact slot: o = x * x (dense, same shape)
      hs.push_back(rt.submit(OpKind::Mul, {x, x}, o));
    } else {
      // extended slot: o = x + consts[i] (rank-0 broadcast view)
      TensorView c = consts;
      c.shape = {};
      c.strides = {};
      c.offset = i;
      hs.push_back(rt.submit(OpKind::Add, {x, c}, o));
    }
  }
  rt.wait_all();
  stop.store(true, std::memory_order_release);
  monitor.join();
  std::printf("  %llu peek samples during the run\n", (unsigned long long)samples.load());
  CHECK(samples.load() > 100);
  CHECK(violations.load() == 0);
  CHECK(regressions.load() == 0);
  uint64_t not_done = 0, xor_want = 0;
  for (const TaskHandle& h : hs) {
    not_done += h.state() == TaskState::Done ? 0 : 1;
    xor_want ^= h.id();
  }
  CHECK(not_done == 0);
  const std::vector<double> got = read_all(rt, out);
  uint64_t bad = 0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < len; ++k) {
      const double want = i % 2 == 0 ? f32(xv[k] * xv[k]) : f32(xv[k] + cv[i]);
      bad += got[static_cast<size_t>(i) * len + k] == want ? 0 : 1;
    }
  CHECK(bad == 0);
  const auto tr = rt.trace();
  REQUIRE(tr.size() == static_cast<size_t>(n));
  std::vector<uint8_t> seen(static_cast<size_t>(n) + 2, 0);
  uint64_t xor_seen = 0, dup = 0, foreign = 0;
  const uint64_t base = hs.front().id();
  for (const Tracepoint& t : tr) {
    xor_seen ^= t.seq;
    if (t.seq < base || t.seq - base >= static_cast<uint64_t>(n)) {
      ++foreign;
      continue;
    }
    dup += seen[t.seq - base]++ ? 1 : 0;
  }
  CHECK(dup == 0);
  CHECK(foreign == 0);
  CHECK(xor_seen == xor_want);
  const CounterSnapshot c = rt.counters();
  CHECK(c.processed == c.committed);
  CHECK(c.committed == static_cast<uint64_t>(n));
  const auto s = rt.peek_queue();
  CHECK(s.processed == s.head);
  CHECK(s.head == s.tail);
}

// Extension (the reference orders work only through host waits): fence()
// makes later tasks wait on the device for every earlier task, so a chain of
// dependent phases runs back to back with a single host wait at the end.
TEST_CASE("fence: dependent phases without host waits match the waited sequence") {
  Runtime rt(small_config(4096, 0));
  const int n = 1500, len = 4096;
  auto x = rt.alloc_tensor(DType::F32, {int64_t{n} * len});
  auto a = rt.alloc_tensor(DType::F32, {int64_t{n} * len});
  auto b = rt.alloc_tensor(DType::F32, {int64_t{n} * len});
  auto c = rt.alloc_tensor(DType::F32, {int64_t{n} * len});
  std::mt19937_64 rng(7);
  std::vector<double> xv = random_vals(rng, static_cast<size_t>(n) * len, -2.0, 2.0);
  for (double& v : xv) v = f32(v);  // the values an f32 buffer holds
  fill(rt, x, xv);
  auto row = [&](const TensorView& base, int i) {
    TensorView v = base;
    v.shape = {len};
    v.strides = {1};
    v.offset = int64_t{i} * len;
    return v;
  };
  std::vector<TaskHandle> hs;
  for (int rep = 0; rep < 3; ++rep) {
    hs.clear();
    for (int i = 0; i < n; ++i) hs.push_back(rt.submit(OpKind::Relu, {row(x, i)}, row(a, i)));
    rt.fence();
    for (int i = 0; i < n; ++i) hs.push_back(rt.submit(OpKind::Mul, {row(a, i), row(x, i)}, row(b, i)));
    rt.fence();
    // extended slots too: a rank-0 broadcast of the previous phase's output
    for (int i = 0; i < n; ++i) {
      TensorView s0 = row(b, (i + 1) % n);
      s0.shape = {};
      s0.strides = {};
      hs.push_back(rt.submit(OpKind::Add, {row(b, i), s0}, row(c, i)));
    }
    rt.wait_all();
    uint64_t bad_state = 0;
    for (const TaskHandle& h : hs) bad_state += h.state() == TaskState::Done ? 0 : 1;
    CHECK(bad_state == 0);
    const std::vector<double> got = read_all(rt, c);
    uint64_t bad = 0;
    for (int i = 0; i < n; ++i) {
      const double x1 = xv[static_cast<size_t>((i + 1) % n) * len];
      const double s0 = f32((x1 < 0 ? 0.0 : x1) * x1);
      for (int k = 0; k < len; ++k) {
        const double xi = xv[static_cast<size_t>(i) * len + k];
        const double ai = xi < 0 ? 0.0 : xi;
        const double bi = f32(ai * xi);
        bad += got[static_cast<size_t>(i) * len + k] == f32(bi + s0) ? 0 : 1;
      }
    }
    CHECK(bad == 0);
    // clear the outputs so the next rep cannot pass on stale values
    fill(rt, a, std::vector<double>(static_cast<size_t>(n) * len, -7.0));
    fill(rt, b, std::vector<double>(static_cast<size_t>(n) * len, -7.0));
    fill(rt, c, std::vector<double>(static_cast<size_t>(n) * len, -7.0));
  }
  const CounterSnapshot cs = rt.counters();
  CHECK(cs.processed == cs.committed);
}

TEST_CASE("hot swap under load: every row is entirely one variant, no canary hits") {
  Runtime rt(small_config(4096, 0));
  const double pa[2] = {1.5, -0.25};
  const double pb[2] = {-2.0, 3.0};
  const uint32_t id = static_cast<uint32_t>(rt.inject_operator("scale_add", pa));
  constexpr int kRows = 8, kN = 4096, kTasks = 20000;
  std::vector<TensorView> ins, outs;
  std::mt19937_64 rng(808);
  std::vector<std::vector<double>> iv;
  for (int r = 0; r < kRows; ++r) {
    ins.push_back(rt.alloc_tensor(DType::F32, {kN}));
    iv.push_back(random_vals(rng, kN, -1.0, 1.0));
    fill(rt, ins.back(), iv.back());
  }
  for (int t = 0; t < kTasks; ++t) outs.push_back(rt.alloc_tensor(DType::F32, {kN}));
  std::vector<TaskHandle> hs;
  hs.reserve(kTasks);
  for (int t = 0; t < kTasks; ++t) {
    hs.push_back(rt.submit(id, {ins[static_cast<size_t>(t % kRows)]}, outs[static_cast<size_t>(t)]));
    if (t == kTasks / 2) rt.inject_operator_at(id, "scale_add", pb);
  }
  rt.wait_all();
  int old_rows = 0, new_rows = 0;
  for (int t = 0; t < kTasks; ++t) {
    REQUIRE(hs[static_cast<size_t>(t)].state() == TaskState::Done);
    const auto got = read_all(rt, outs[static_cast<size_t>(t)]);
    const auto& x = iv[static_cast<size_t>(t % kRows)];
    bool all_a = true, all_b = true;
    for (int e = 0; e < kN; ++e) {
      const double xv = f32(x[static_cast<size_t>(e)]);
      all_a = all_a && got[static_cast<size_t>(e)] == f32(xv * 1.5 + -0.25);
      all_b = all_b && got[static_cast<size_t>(e)] == f32(xv * -2.0 + 3.0);
    }
    REQUIRE((all_a || all_b));
    (all_a ? old_rows : new_rows) += 1;
    if (t > kTasks / 2 + 2 * 4096) CHECK(all_b);  // past the ring's in-flight window
  }
  CHECK(old_rows > 0);
  CHECK(new_rows > 0);
  CHECK(rt.canary_hits() == 0);
  const gpuos_inject_stats& st = rt.last_inject_stats();
  std::printf("  swap: upload %.1f us, epoch wait %.1f us, bank write %.1f us, flip %.1f us; rows old=%d new=%d\n",
              st.upload_ns / 1e3, st.epoch_wait_ns / 1e3, st.bank_write_ns / 1e3, st.flip_ns / 1e3, old_rows, new_rows);
}

TEST_CASE("native promotion: NVRTC + nvJitLink op, generation handover, bit-identical to the program") {
  Runtime rt(small_config(4096, 0));
  std::mt19937_64 rng(909);
  const double pa[2] = {1.5, -0.25};
  // every shipped template, f32 and f64: the native code must return exactly
  // what the device program returns (and what eval_expr + narrow gives)
  const std::vector<std::string> names = rt.templates().names();
  struct Op {
    uint64_t id;
    int arity;
    DType dt;
  };
  std::vector<Op> ops;
  for (const std::string& name : names)
    for (DType dt : {DType::F32, DType::F64}) {
      const OperatorTemplate t = rt.templates().get(name);
      const double params[8] = {0.75, 2.5, 0, 0, 0, 0, 0, 0};
      ops.push_back({rt.inject_operator(name, params, dt), t.arity, dt});
    }
  const uint64_t sa = rt.inject_operator("scale_add", pa);
  ops.push_back({sa, 1, DType::F32});
  const int64_t n = 3000;  // ragged: not a multiple of the vector width
  std::vector<std::vector<TensorView>> ins(ops.size());
  std::vector<TensorView> out_prog, out_nat;
  for (size_t i = 0; i < ops.size(); ++i) {
    for (int k = 0; k < ops[i].arity; ++k) {
      ins[i].push_back(rt.alloc_tensor(ops[i].dt, {n}));
      fill(rt, ins[i].back(), random_vals(rng, static_cast<size_t>(n), -3.0, 3.0));
    }
    out_prog.push_back(rt.alloc_tensor(ops[i].dt, {n}));
    out_nat.push_back(rt.alloc_tensor(ops[i].dt, {n}));
    REQUIRE(rt.wait(rt.submit(ops[i].id, ins[i], out_prog[i])) == TaskState::Done);
  }
  double compile_ms = 0, link_ms = 0, handover_us = 0;
  for (size_t i = 0; i < ops.size(); ++i) {
    rt.promote_native(static_cast<uint32_t>(ops[i].id));
    const auto& st = rt.last_native_stats();
    compile_ms += st.compile_ns / 1e6;
    link_ms = st.link_ns / 1e6;
    handover_us = (st.handover.drain_ns + st.handover.load_ns + st.handover.relaunch_ns) / 1e3;
    REQUIRE(rt.is_native(static_cast<uint32_t>(ops[i].id)));
  }
  REQUIRE(rt.worker_alive());
  for (size_t i = 0; i < ops.size(); ++i) {
    REQUIRE(rt.wait(rt.submit(ops[i].id, ins[i], out_nat[i])) == TaskState::Done);
    REQUIRE(read_all(rt, out_nat[i]) == read_all(rt, out_prog[i]));
  }
  // strided + broadcast operands through the native body
  auto bx = rt.alloc_tensor(DType::F32, {8, 64});
  fill(rt, bx, random_vals(rng, 8 * 64));
  TensorView row = bx;
  row.shape = {1, 64};
  row.strides = {64, 1};
  auto bo = rt.alloc_tensor(DType::F32, {16, 64});
  REQUIRE(rt.wait(rt.submit(sa, {row}, bo)) == TaskState::Done);
  const auto xv = read_all(rt, bx);
  const auto bov = read_all(rt, bo);
  for (int r = 0; r < 16; ++r)
    for (int c = 0; c < 64; ++c) REQUIRE(bov[static_cast<size_t>(r * 64 + c)] == f32(xv[static_cast<size_t>(c)] * 1.5 + -0.25));
  // errors keep the program's codes
  auto o64 = rt.alloc_tensor(DType::F64, {n});
  auto he = rt.submit(sa, {ins.back()[0]}, o64);
  REQUIRE(rt.wait(he) == TaskState::Failed);
  CHECK(he.error() == ErrorCode::DTypeMismatch);
  CHECK(rt.canary_hits() == 0);
  std::printf("  native: %zu ops, nvrtc %.1f ms total, last nvJitLink %.1f ms, last handover %.1f us\n", ops.size(),
              compile_ms, link_ms, handover_us);
}

TEST_CASE("fusion: composites equal the waited sequential run; retained steps materialize") {
  for (DType dt : {DType::F32, DType::F64}) {
    Runtime rt(small_config(4096, 0));
    const double pa[2] = {1.5, -0.25};
    const uint64_t sa = rt.inject_operator("scale_add", pa, dt);
    std::mt19937_64 rng(4242);
    const int64_t n = 4096;
    auto x = rt.alloc_tensor(dt, {n});
    auto y = rt.alloc_tensor(dt, {n});
    fill(rt, x, random_vals(rng, static_cast<size_t>(n), -2.0, 2.0));
    fill(rt, y, random_vals(rng, static_cast<size_t>(n), -2.0, 2.0));
    // chain: t1 = x + y; t2 = t1 * x; t3 = relu(t2); t4 = gelu(t3); t5 = scale_add(t4)
    auto run_chain = [&](bool fused, std::vector<TensorView>& t, bool keep_t2) {
      for (int k = 0; k < 5; ++k) t.push_back(rt.alloc_tensor(dt, {n}));
      rt.set_fusion(fused);
      std::vector<TaskHandle> keep;
      auto step = [&](uint64_t op, std::vector<TensorView> ins, const TensorView& o, bool hold) {
        TaskHandle h = rt.submit(op, std::move(ins), o);
        if (!fused) REQUIRE(rt.wait(h) == TaskState::Done);  // waited sequential
        if (hold) keep.push_back(h);
      };
      step(static_cast<uint64_t>(OpKind::Add), {x, y}, t[0], false);
      step(static_cast<uint64_t>(OpKind::Mul), {t[0], x}, t[1], keep_t2);
      step(static_cast<uint64_t>(OpKind::Relu), {t[1]}, t[2], false);
      step(static_cast<uint64_t>(OpKind::Gelu), {t[2]}, t[3], false);
      step(sa, {t[3]}, t[4], true);
      for (const TaskHandle& h : keep) REQUIRE(rt.wait(h) == TaskState::Done);
      rt.set_fusion(false);
    };
    std::vector<TensorView> seq, fus, fus2;
    run_chain(false, seq, false);
    const uint64_t absorbed0 = rt.fusion_absorbed();
    run_chain(true, fus, false);
    CHECK(rt.fusion_absorbed() - absorbed0 == 4);  // five steps behind one descriptor
    REQUIRE(read_all(rt, fus[4]) == read_all(rt, seq[4]));
    // a retained handle splits the chain and materializes its output
    run_chain(true, fus2, true);
    REQUIRE(read_all(rt, fus2[1]) == read_all(rt, seq[1]));
    REQUIRE(read_all(rt, fus2[4]) == read_all(rt, seq[4]));
    // fuse(calls): every returned handle completes; the chain's tail is exact
    std::vector<TensorView> t;
    for (int k = 0; k < 3; ++k) t.push_back(rt.alloc_tensor(dt, {n}));
    std::vector<OpCall> calls(3);
    calls[0] = OpCall{static_cast<uint64_t>(OpKind::Add), {x, y}, t[0], {}};
    calls[1] = OpCall{static_cast<uint64_t>(OpKind::Mul), {t[0], x}, t[1], {}};
    calls[2] = OpCall{static_cast<uint64_t>(OpKind::Relu), {t[1]}, t[2], {}};
    const std::vector<TaskHandle> hs = rt.fuse(calls);
    for (const TaskHandle& h : hs) REQUIRE(rt.wait(h) == TaskState::Done);
    REQUIRE(read_all(rt, t[2]) == read_all(rt, seq[2]));
    rt.wait_all();
    const CounterSnapshot c = rt.counters();
    CHECK(c.submitted == c.inline_executions + c.committed + rt.fusion_absorbed());  // runtime.hpp:325-327
    CHECK(rt.canary_hits() == 0);
  }
}

// Fused composites against the oracle (not only against the device's own
// sequential run): the chain add -> mul -> relu -> gelu, fused into one
// composite, equals the oracle (oracle/liboracle.so, the C restatement pinned
// to the reference) applied step by step with each step narrowed to the
// dtype: bit-exact through relu, gelu within its stated tolerance
// (rel 1e-6 f32, 1e-12 f64: the device's tanh is not glibc's).
TEST_CASE("fusion: fused chains equal the oracle applied step by step") {
  std::string exe(4096, '\0');
  const ssize_t len = readlink("/proc/self/exe", exe.data(), exe.size() - 1);
  REQUIRE(len > 0);
  exe.resize(static_cast<size_t>(len));
  const std::string root = exe.substr(0, exe.rfind("/build/"));
  REQUIRE(gbcheck::load_oracle((root + "/oracle/liboracle.so").c_str()));
  const gbcheck::Oracle& O = gbcheck::oracle();
  for (DType dt : {DType::F32, DType::F64}) {
    Runtime rt(small_config(4096, 0));
    const int64_t n = 4096;
    std::mt19937_64 rng(99);
    auto x = rt.alloc_tensor(dt, {n});
    auto y = rt.alloc_tensor(dt, {n});
    std::vector<double> xv = random_vals(rng, static_cast<size_t>(n), -2.0, 2.0);
    std::vector<double> yv = random_vals(rng, static_cast<size_t>(n), -2.0, 2.0);
    if (dt == DType::F32)
      for (auto* v : {&xv, &yv})
        for (double& e : *v) e = f32(e);
    fill(rt, x, xv);
    fill(rt, y, yv);
    std::vector<TensorView> t;
    for (int k = 0; k < 4; ++k) t.push_back(rt.alloc_tensor(dt, {n}));
    rt.set_fusion(true);
    rt.submit(OpKind::Add, {x, y}, t[0]);
    rt.submit(OpKind::Mul, {t[0], x}, t[1]);
    rt.submit(OpKind::Relu, {t[1]}, t[2]);
    TaskHandle last = rt.submit(OpKind::Gelu, {t[2]}, t[3]);
    REQUIRE(rt.wait(last) == TaskState::Done);
    rt.set_fusion(false);
    CHECK(rt.fusion_absorbed() == 3);
    const std::vector<double> got = read_all(rt, t[3]);
    // oracle, step by step, each output narrowed to dt
    const int odt = dt == DType::F32 ? ORC_F32 : ORC_F64;
    const size_t w = dt == DType::F32 ? 4 : 8;
    std::vector<unsigned char> hx(static_cast<size_t>(n) * w), hy(hx.size()), s1(hx.size()), s2(hx.size()),
        s3(hx.size()), s4(hx.size());
    for (int64_t i = 0; i < n; ++i) {
      if (dt == DType::F32) {
        const float a = static_cast<float>(xv[i]), b = static_cast<float>(yv[i]);
        std::memcpy(&hx[i * 4], &a, 4);
        std::memcpy(&hy[i * 4], &b, 4);
      } else {
        std::memcpy(&hx[i * 8], &xv[i], 8);
        std::memcpy(&hy[i * 8], &yv[i], 8);
      }
    }
    auto v = [&](std::vector<unsigned char>& b) { return gbcheck::view(b.data(), odt, 0, {n}, {1}); };
    orc_view o1 = v(s1), o2 = v(s2), o3 = v(s3), o4 = v(s4), vx = v(hx), vy = v(hy);
    orc_view in01[2] = {vx, vy};
    REQUIRE(O.elementwise(0, &o1, in01, 2) == 0);
    orc_view in12[2] = {o1, vx};
    REQUIRE(O.elementwise(1, &o2, in12, 2) == 0);
    REQUIRE(O.elementwise(2, &o3, &o2, 1) == 0);
    REQUIRE(O.elementwise(3, &o4, &o3, 1) == 0);
    // the intermediate steps were elided on the device; the chain's input to
    // gelu must match the oracle exactly, so compare relu(...) through a
    // materialized run as well
    const double tol = dt == DType::F32 ? 1e-6 : 1e-12;
    uint64_t bad = 0, exact = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double want = gbcheck::decode(odt, s4.data(), i);
      exact += got[static_cast<size_t>(i)] == want ? 1 : 0;
      if (!close_tol(got[static_cast<size_t>(i)], want, tol)) ++bad;
    }
    std::printf("  %s: %llu/%lld gelu outputs bit-identical to the oracle, %llu outside tolerance\n",
                dt == DType::F32 ? "f32" : "f64", (unsigned long long)exact, (long long)n, (unsigned long long)bad);
    CHECK(bad == 0);
    // a retained handle materializes its step: bit-exact against the oracle
    std::vector<TensorView> u;
    for (int k = 0; k < 3; ++k) u.push_back(rt.alloc_tensor(dt, {n}));
    rt.set_fusion(true);
    rt.submit(OpKind::Add, {x, y}, u[0]);
    TaskHandle keep = rt.submit(OpKind::Mul, {u[0], x}, u[1]);
    TaskHandle tail = rt.submit(OpKind::Relu, {u[1]}, u[2]);
    REQUIRE(rt.wait(tail) == TaskState::Done);
    REQUIRE(rt.wait(keep) == TaskState::Done);
    rt.set_fusion(false);
    const std::vector<double> g1 = read_all(rt, u[1]), g2 = read_all(rt, u[2]);
    uint64_t bad_exact = 0;
    for (int64_t i = 0; i < n; ++i) {
      bad_exact += g1[static_cast<size_t>(i)] == gbcheck::decode(odt, s2.data(), i) ? 0 : 1;
      bad_exact += g2[static_cast<size_t>(i)] == gbcheck::decode(odt, s3.data(), i) ? 0 : 1;
    }
    CHECK(bad_exact == 0);
  }
}

// The reference's producer-side TaskQueue API (queue.hpp:156-300) over the
// device ring: acquire_slot / commit / peek / wait_for_processed, with the
// persistent workers as the consumer (try_claim / mark_done on the device).
TEST_CASE("TaskQueue producer API: acquire, commit, peek over the device ring") {
  Runtime rt(small_config(64, 4));
  const int64_t n = 1000;
  auto x = rt.alloc_tensor(DType::F32, {n});
  auto y = rt.alloc_tensor(DType::F32, {n});
  std::vector<double> xv(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) xv[static_cast<size_t>(i)] = static_cast<double>(i % 17) - 8.0;
  fill(rt, x, xv);
  rt.wait_all();
  TaskQueue q(rt.device());
  CHECK(q.capacity() == 64);
  const TaskQueue::Snapshot s0 = q.peek();
  gpuos_task t;
  std::memset(&t, 0, sizeof(t));
  t.op_id = static_cast<uint32_t>(OpKind::Relu);
  t.n_inputs = 1;
  t.size = static_cast<uint64_t>(n);
  const auto view_of = [&](const TensorView& v, gpuos_view* o) {
    o->addr = reinterpret_cast<uint64_t>(rt.pool().lookup(v.buffer).data);
    o->extents[0] = static_cast<int32_t>(n);
    o->strides[0] = 1;
    o->dtype = GPUOS_F32;
    o->rank = 1;
    o->status = GPUOS_VIEW_OK;
  };
  view_of(y, &t.views[0]);
  view_of(x, &t.views[1]);
  const int tasks = 200;  // > capacity: acquire_slot reports a full ring until workers free slots
  uint64_t full = 0;
  for (int i = 0; i < tasks; ++i) {
    t.seq = 900000 + static_cast<uint64_t>(i);
    std::optional<uint64_t> pos;
    while (!(pos = q.acquire_slot())) ++full;
    q.commit(*pos, t);
  }
  REQUIRE(q.wait_for_processed(s0.processed + tasks) == 0);
  const TaskQueue::Snapshot s1 = q.peek();
  CHECK(s1.tail - s0.tail == static_cast<uint64_t>(tasks));
  CHECK(s1.processed == s1.head);
  CHECK(s1.head == s1.tail);
  const std::vector<double> got = read_all(rt, y);
  uint64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) bad += got[static_cast<size_t>(i)] == std::max(0.0, xv[static_cast<size_t>(i)]) ? 0 : 1;
  CHECK(bad == 0);
  std::printf("  %d tasks through TaskQueue, %llu full-ring retries\n", tasks, (unsigned long long)full);
}

TEST_CASE("shutdown drains every committed task") {
  Runtime rt(small_config(1024, 0));
  auto x = rt.alloc_tensor(DType::F32, {256});
  auto y = rt.alloc_tensor(DType::F32, {256});
  std::vector<TaskHandle> hs;
  for (int i = 0; i < 10000; ++i) hs.push_back(rt.submit(OpKind::Relu, {x}, y));
  rt.shutdown();
  for (const TaskHandle& h : hs) REQUIRE(h.state() == TaskState::Done);
  REQUIRE_FALSE(rt.worker_alive());
}

TEST_CASE("kv_append writes the row and reports CacheFull past capacity") {
  Runtime rt(small_config());
  const int64_t h = 2, cap = 4, d = 8;
  auto kc = rt.alloc_tensor(DType::F32, {h, cap, d});
  auto vc = rt.alloc_tensor(DType::F32, {h, cap, d});
  auto nk = rt.alloc_tensor(DType::F32, {h, d});
  auto nv = rt.alloc_tensor(DType::F32, {h, d});
  std::mt19937_64 rng(909);
  const auto wk = random_vals(rng, static_cast<size_t>(h * d)), wv = random_vals(rng, static_cast<size_t>(h * d));
  fill(rt, nk, wk);
  fill(rt, nv, wv);
  for (int64_t cur = 0; cur < cap; ++cur)
    REQUIRE(rt.wait(rt.submit(OpKind::KvAppend, {nk, nv, vc}, kc, {static_cast<double>(cur)})) == TaskState::Done);
  BoundView bk(rt.pool(), kc), bv(rt.pool(), vc);
  for (int64_t hh = 0; hh < h; ++hh)
    for (int64_t cur = 0; cur < cap; ++cur)
      for (int64_t e = 0; e < d; ++e) {
        REQUIRE(bk.load((hh * cap + cur) * d + e) == f32(wk[static_cast<size_t>(hh * d + e)]));
        REQUIRE(bv.load((hh * cap + cur) * d + e) == f32(wv[static_cast<size_t>(hh * d + e)]));
      }
  auto bad = rt.submit(OpKind::KvAppend, {nk, nv, vc}, kc, {static_cast<double>(cap)});
  REQUIRE(rt.wait(bad) == TaskState::Failed);
  REQUIRE(bad.error() == ErrorCode::CacheFull);
}

TEST_CASE("telemetry: tracepoints per dispatch, CSV and JSONL round trip") {
  Runtime rt(small_config());
  auto x = rt.alloc_tensor(DType::F32, {64});
  auto y = rt.alloc_tensor(DType::F32, {64});
  for (int i = 0; i < 100; ++i) rt.submit(OpKind::Relu, {x}, y);
  rt.wait_all();
  const auto tr = rt.trace();
  REQUIRE(tr.size() == 100);
  for (const Tracepoint& t : tr) {
    CHECK(t.dequeue_ns >= t.enqueue_ns);
    CHECK(t.exec_ns >= 1);
    CHECK(t.op_id == static_cast<uint64_t>(OpKind::Relu));
  }
  std::stringstream cs, js;
  export_csv(tr, cs);
  export_jsonl(tr, js);
  CHECK(parse_trace_csv(cs) == tr);
  CHECK(parse_trace_jsonl(js) == tr);
  const auto lat = latency_ns(tr);
  std::printf("  queue latency p50 %llu ns p99 %llu ns\n", (unsigned long long)percentile(lat, 0.5),
              (unsigned long long)percentile(lat, 0.99));
}
