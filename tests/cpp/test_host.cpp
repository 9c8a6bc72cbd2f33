// Host-logic suite (no GPU): restates the CPU-side reference tests —
// test_tensor.cpp, the parser / lowering / verifier / cache / registry parts of
// test_opcompiler.cpp and the export half of test_telemetry.cpp — against the
// B200 build's headers, plus the new F16/BF16 storage and small-vector shape.
#include <gpuos/bytecode.hpp>
#include <gpuos/expr.hpp>
#include <gpuos/opcompiler.hpp>
#include <gpuos/optable.hpp>
#include <gpuos/telemetry.hpp>
#include <gpuos/tensor.hpp>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <random>
#include <sstream>
#include <thread>

#include "check.hpp"

using namespace gpuos;

namespace {

bool same_value(double a, double b) { return (std::isnan(a) && std::isnan(b)) || a == b; }

// Reference-free random AST generator (the idea of test_opcompiler.cpp:66-99).
ExprPtr gen_expr(std::mt19937& rng, int depth, int arity, int n_params) {
  std::uniform_int_distribution<int> pick(0, depth > 0 ? 9 : 2);
  const int k = pick(rng);
  if (k == 0 || (k == 1 && arity == 0)) return make_const(std::uniform_real_distribution<double>(-4, 4)(rng));
  if (k == 1) return make_in(std::uniform_int_distribution<int>(0, arity - 1)(rng));
  if (k == 2) return make_param(std::uniform_int_distribution<int>(0, n_params - 1)(rng));
  static const ExprKind un[] = {ExprKind::Neg, ExprKind::Exp, ExprKind::Tanh, ExprKind::Abs, ExprKind::Sqrt};
  static const ExprKind bi[] = {ExprKind::Add, ExprKind::Sub, ExprKind::Mul, ExprKind::Div, ExprKind::Max,
                                ExprKind::Min};
  if (k <= 4) return make_unary(un[std::uniform_int_distribution<int>(0, 4)(rng)], gen_expr(rng, depth - 1, arity, n_params));
  return make_binary(bi[std::uniform_int_distribution<int>(0, 5)(rng)], gen_expr(rng, depth - 1, arity, n_params),
                     gen_expr(rng, depth - 1, arity, n_params));
}

int max_depth_run(const Bytecode& code) {
  int d = 0, hi = 0;
  for (const Instr& i : code) {
    if (i.op == OpCode::PushConst || i.op == OpCode::LoadIn) ++d;
    else if (i.op == OpCode::Add || i.op == OpCode::Sub || i.op == OpCode::Mul || i.op == OpCode::Div ||
             i.op == OpCode::Max || i.op == OpCode::Min || i.op == OpCode::StoreOut)
      --d;
    hi = std::max(hi, d);
  }
  return hi;
}

}  // namespace

TEST_CASE("dtype widths and names") {
  CHECK(dtype_width(DType::F32) == 4);
  CHECK(dtype_width(DType::F64) == 8);
  CHECK(dtype_width(DType::I32) == 4);
  CHECK(dtype_width(DType::F16) == 2);
  CHECK(dtype_width(DType::BF16) == 2);
  CHECK(std::string(dtype_name(DType::BF16)) == "bf16");
}

TEST_CASE("contiguous strides, broadcast, element offsets") {
  CHECK(contiguous_strides(Shape{2, 3}) == (Strides{3, 1}));
  CHECK(contiguous_strides(Shape{}) == Strides{});
  CHECK(contiguous_strides(Shape{4, 1, 5}) == (Strides{5, 5, 1}));
  CHECK(broadcast_shapes(Shape{3, 1}, Shape{1, 4}) == (Shape{3, 4}));
  CHECK_THROWS_AS(broadcast_shapes(Shape{2, 3}, Shape{4, 3}), Error);
  TensorView v;
  v.buffer = 42;
  v.shape = {3, 1};
  v.strides = {1, 1};
  TensorView b = broadcast_view(v, Shape{3, 4});
  CHECK(b.buffer == 42);
  CHECK(b.strides == (Strides{1, 0}));
  TensorView scalar;
  CHECK(broadcast_view(scalar, Shape{2, 2}).strides == (Strides{0, 0}));
  TensorView w;
  w.shape = {2, 3};
  w.strides = {3, 1};
  CHECK(element_offset(w, {1, 2}) == 5);
  TensorView x;
  x.offset = 10;
  x.shape = {8, 3};
  x.strides = {0, 1};
  CHECK(element_offset(x, {7, 2}) == 12);
  CHECK_THROWS_AS(element_offset(w, {2, 0}), Error);
  TensorView r;
  r.offset = 4;
  r.shape = {5};
  r.strides = {-1};
  for (int64_t i = 0; i < 5; ++i) CHECK(element_offset(r, {i}) == 4 - i);
  // symmetric broadcast over random shapes
  std::mt19937 rng(7002);
  for (int t = 0; t < 200; ++t) {
    Shape a, c;
    for (int i = std::uniform_int_distribution<int>(0, 4)(rng); i > 0; --i) a.push_back(std::uniform_int_distribution<int>(1, 3)(rng));
    for (int i = std::uniform_int_distribution<int>(0, 4)(rng); i > 0; --i) c.push_back(std::uniform_int_distribution<int>(1, 3)(rng));
    bool ok1 = true, ok2 = true;
    Shape ab, ba;
    try { ab = broadcast_shapes(a, c); } catch (const Error&) { ok1 = false; }
    try { ba = broadcast_shapes(c, a); } catch (const Error&) { ok2 = false; }
    CHECK(ok1 == ok2);
    if (ok1) CHECK(ab == ba);
  }
}

TEST_CASE("Dims behaves like the reference's vector shapes") {
  Dims d{1, 2, 3, 4, 5, 6, 7, 8};  // spills past the inline capacity
  CHECK(d.size() == 8);
  CHECK(d[7] == 8);
  Dims e = d;
  CHECK(e == d);
  e.pop_back();
  CHECK(e != d);
  CHECK(shape_to_string(e) == "(1,2,3,4,5,6,7)");
  std::vector<int64_t> as_vec = d;
  CHECK(as_vec.size() == 8);
  Dims f(std::move(e));
  CHECK(f.size() == 7);
  CHECK(e.empty());
}

TEST_CASE("host BufferPool: zero-filled, never-reused ids, release rules") {
  BufferPool pool;
  const BufferId a = pool.allocate(DType::F32, 8);
  const BufferId b = pool.allocate(DType::F64, 0);
  CHECK(a != b);
  for (int i = 0; i < 8; ++i) CHECK(pool.data<float>(a)[i] == 0.0f);
  pool.release(a);
  CHECK_FALSE(pool.contains(a));
  CHECK_THROWS_AS(pool.release(a), Error);
  CHECK_THROWS_AS(pool.lookup(a), Error);
  const BufferId c = pool.allocate(DType::F32, 8);
  CHECK(c != a);
  CHECK(pool.size() == 2);
}

TEST_CASE("BoundView narrows once on store, including f16/bf16") {
  BufferPool pool;
  for (DType dt : {DType::F32, DType::F64, DType::I32, DType::F16, DType::BF16}) {
    TensorView v;
    v.dtype = dt;
    v.shape = {4};
    v.strides = {1};
    v.buffer = pool.allocate(dt, 4);
    BoundView bv(pool, v);
    const double vals[4] = {1.0 / 3.0, -2.5, 65504.0, 1e-7};
    for (int i = 0; i < 4; ++i) bv.store(i, vals[i]);
    for (int i = 0; i < 4; ++i) CHECK(bv.load(i) == narrow_to(dt, vals[i]));
  }
  CHECK(bf16_from_double(1.0 + std::ldexp(1.0, -8) + std::ldexp(1.0, -30)) == 0x3F81);
  CHECK(f16_from_double(65520.0) == 0x7C00);
  CHECK(narrow_i32(3e9) == INT32_MIN);
  TensorView wrong;
  wrong.dtype = DType::F64;
  wrong.buffer = pool.allocate(DType::F32, 1);
  CHECK_THROWS_AS(BoundView(pool, wrong), Error);
}

TEST_CASE("IndexIterator walks row-major with per-operand offsets") {
  TensorView a, b;
  a.shape = {2, 3};
  a.strides = {3, 1};
  b.shape = {2, 3};
  b.strides = {1, 2};
  b.offset = 1;
  const TensorView* ops[] = {&a, &b};
  IndexIterator it(a.shape, ops);
  std::vector<int64_t> oa, ob;
  for (int64_t i = 0; i < it.count(); ++i, it.next()) {
    oa.push_back(it.offset(0));
    ob.push_back(it.offset(1));
  }
  CHECK(oa == (std::vector<int64_t>{0, 1, 2, 3, 4, 5}));
  CHECK(ob == (std::vector<int64_t>{1, 3, 5, 2, 4, 6}));
}

TEST_CASE("parser builds trees, prints re-parseably, reports errors with positions") {
  ExprPtr sum = parse_expression("in0 + in1");
  REQUIRE(sum->kind == ExprKind::Add);
  CHECK(sum->b->index == 1);
  ExprPtr aff = parse_expression("in0 * $p0 + $p1");
  CHECK(aff->a->kind == ExprKind::Mul);
  CHECK(aff->b->kind == ExprKind::Param);
  for (const char* src : {"in0 + in1", "max(in0, 0)", "1 / (1 + exp(-in0))", "min(max(in0, $p0), $p1)",
                          "abs(in0 - in1) * sqrt(in2)", "-in0 * -2.5e-2 + tanh($p7)", "3.25"}) {
    ExprPtr a = parse_expression(src);
    ExprPtr b = parse_expression(expr_to_string(*a));
    CHECK(expr_equal(*a, *b));
  }
  auto code_of = [](const char* s) {
    try {
      parse_expression(s);
    } catch (const Error& e) {
      return e.code();
    }
    return ErrorCode::Ok;
  };
  CHECK(code_of("in0 +") == ErrorCode::SyntaxError);
  CHECK(code_of("(in0") == ErrorCode::SyntaxError);
  CHECK(code_of("in0 in1") == ErrorCode::SyntaxError);
  CHECK(code_of("$q0") == ErrorCode::SyntaxError);
  CHECK(code_of("foo") == ErrorCode::UnknownIdentifier);
  CHECK(code_of("foo(in0)") == ErrorCode::UnknownIdentifier);
  CHECK(code_of("in7") == ErrorCode::UnknownIdentifier);
  CHECK(code_of("$p9") == ErrorCode::UnknownIdentifier);
  CHECK(code_of("exp(in0, in1)") == ErrorCode::ArityError);
  CHECK(code_of("max(in0)") == ErrorCode::ArityError);
  try {
    parse_expression("in0 + @");
    CHECK(false);
  } catch (const Error& e) {
    CHECK(std::string(e.what()).find("at 6") != std::string::npos);
  }
}

TEST_CASE("lowering, verification bounds, interpreter == recursive evaluation") {
  Bytecode code = lower(*parse_expression("in0 + in1"), {});
  REQUIRE(code.size() == 4);
  CHECK(code[0].op == OpCode::LoadIn);
  CHECK(code[2].op == OpCode::Add);
  CHECK(code[3].op == OpCode::StoreOut);
  const double params[8] = {2.0, 3.0, 0, 0, 0, 0, 0, 0};
  Bytecode aff = lower(*parse_expression("in0 * $p0 + $p1"), params);
  CHECK(verify(aff, 1) == 2);
  double stack[16];
  const double four = 4.0;
  CHECK(run_bytecode(aff, {&four, 1}, stack) == 11.0);
  CHECK_THROWS_AS(verify({{OpCode::Add, 0, 0.0}, {OpCode::StoreOut, 0, 0.0}}, 2), Error);
  CHECK_THROWS_AS(verify({{OpCode::PushConst, 0, 1.0}, {OpCode::PushConst, 0, 2.0}, {OpCode::StoreOut, 0, 0.0}}, 0), Error);
  CHECK_THROWS_AS(verify({{OpCode::PushConst, 0, 1.0}}, 0), Error);
  CHECK_THROWS_AS(verify({{OpCode::LoadIn, 2, 0.0}, {OpCode::StoreOut, 0, 0.0}}, 2), Error);
  CHECK_THROWS_AS(lower(*parse_expression("$p3"), std::span<const double>(params, 2)), Error);
  std::mt19937 rng(9002);
  std::uniform_real_distribution<double> dist(-8.0, 8.0);
  for (int trial = 0; trial < 300; ++trial) {
    const int arity = std::uniform_int_distribution<int>(0, 4)(rng);
    double p[8];
    for (double& x : p) x = dist(rng);
    ExprPtr e = gen_expr(rng, std::uniform_int_distribution<int>(0, 5)(rng), arity, 8);
    Bytecode c = lower(*e, p);
    const int ms = verify(c, arity);
    CHECK(ms == max_depth_run(c));
    double in[4];
    for (double& v : in) v = dist(rng);
    CHECK(same_value(run_bytecode(c, {in, 4}, stack), eval_expr(*e, {in, 4}, p)));
  }
}

TEST_CASE("template lowering equals the reference's lowering (tests/golden/programs.json)") {
  const char* path = std::getenv("GPUOS_GOLDEN");
  REQUIRE(path != nullptr);
  std::ifstream f(path);
  REQUIRE(f.good());
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string js = ss.str();
  TemplateRegistry reg = TemplateRegistry::with_defaults();
  const double params[8] = {0.75, 2.5, 0, 0, 0, 0, 0, 0};
  for (const std::string& name : reg.names()) {
    const OperatorTemplate t = reg.get(name);
    const Bytecode code = lower(*substitute_params(*parse_expression(t.source), params), {});
    // serialize like the fixture: [[op, k, value], ...] and compare numerically
    const size_t at = js.find("\"" + name + "\"");
    REQUIRE(at != std::string::npos);
    const size_t cs = js.find("\"code\"", at);
    size_t p = js.find('[', cs) + 1;
    std::vector<double> nums;
    const size_t end = js.find("\"max_stack\"", cs);
    while (p < end) {
      if ((js[p] >= '0' && js[p] <= '9') || js[p] == '-') {
        char* e = nullptr;
        nums.push_back(std::strtod(js.c_str() + p, &e));
        p = static_cast<size_t>(e - js.c_str());
      } else {
        ++p;
      }
    }
    REQUIRE(nums.size() == 3 * code.size());
    for (size_t i = 0; i < code.size(); ++i) {
      CHECK(static_cast<double>(code[i].op) == nums[3 * i]);
      CHECK(static_cast<double>(code[i].k) == nums[3 * i + 1]);
      CHECK(code[i].value == nums[3 * i + 2]);
    }
  }
}

TEST_CASE("module cache: keys include params and dtype, single flight, failures cached") {
  ModuleCache cache;
  OperatorTemplate t{"scale_add", "in0 * $p0 + $p1", 1};
  const double p1[] = {2.0, 1.0}, p2[] = {3.0, 1.0};
  ModulePtr a = cache.compile_or_get(t, p1, DType::F32);
  ModulePtr b = cache.compile_or_get(t, p1, DType::F32);
  CHECK(a.get() == b.get());
  CHECK(cache.hits() == 1);
  CHECK(cache.compile_or_get(t, p2, DType::F32).get() != a.get());
  CHECK(cache.compile_or_get(t, p1, DType::F64).get() != a.get());
  CHECK(cache.compiles() == 3);
  ModuleCache c2;
  OperatorTemplate s{"sigmoid", "1 / (1 + exp(-in0))", 1};
  std::vector<std::thread> ths;
  std::vector<ModulePtr> res(64);
  std::atomic<bool> go{false};
  for (int i = 0; i < 64; ++i)
    ths.emplace_back([&, i] {
      while (!go.load()) std::this_thread::yield();
      res[static_cast<size_t>(i)] = c2.compile_or_get(s, {}, DType::F32);
    });
  go = true;
  for (auto& th : ths) th.join();
  CHECK(c2.compiles() == 1);
  CHECK(c2.hits() == 63);
  OperatorTemplate bad{"bad", "in0 +", 1};
  CHECK_THROWS_AS(c2.compile_or_get(bad, {}, DType::F32), Error);
  CHECK_THROWS_AS(c2.compile_or_get(bad, {}, DType::F32), Error);
  CHECK(c2.misses() == 2);
  OperatorSignature sig;
  sig.template_name = "x";
  sig.params[0] = 0.1;
  CHECK(signature_key(sig) == "x|0.10000000000000001,0,0,0,0,0,0,0|f32|0");
}

TEST_CASE("template registry: defaults, block files, validation") {
  TemplateRegistry r = TemplateRegistry::with_defaults();
  CHECK(r.names().size() == 9);
  std::istringstream good("# comment\n\ntemplate twice arity 1\nexpr: in0 * 2\n\ntemplate mix arity 2\n  expr:  in0 - in1 \n");
  r.load_stream(good);
  CHECK(r.get("mix").source == "in0 - in1");
  std::istringstream bad("template broken arity 1\nnot an expr line\n");
  CHECK_THROWS_AS(r.load_stream(bad), Error);
  CHECK_THROWS_AS(r.add({"too_far", "in1", 1}), Error);
  CHECK_THROWS_AS(r.get("missing"), Error);
  CHECK_THROWS_AS(r.load_file("/nonexistent/templates.txt"), Error);
}

TEST_CASE("telemetry export round trips and nearest-rank percentile") {
  std::vector<Tracepoint> tr;
  for (uint64_t i = 0; i < 50; ++i)
    tr.push_back(Tracepoint{i + 1, i % 14, static_cast<uint32_t>(i % 3), 1000 + i, 1500 + 2 * i, 7 + i, 15});
  tr.back().worker = 0xFFFFFFFFu;
  std::stringstream cs, js;
  CHECK(export_csv(tr, cs) == 50);
  CHECK(export_jsonl(tr, js) == 50);
  CHECK(parse_trace_csv(cs) == tr);
  CHECK(parse_trace_jsonl(js) == tr);
  std::istringstream bad("nope\n1,2,3\n");
  CHECK_THROWS_AS(parse_trace_csv(bad), Error);
  const auto lat = latency_ns(tr);
  CHECK(lat.front() == 500);
  CHECK(percentile(lat, 0.0) == lat.front());
  CHECK(percentile(lat, 1.0) == lat.back());
  CHECK(percentile({1, 2, 3, 4}, 0.5) == 3);
  std::istringstream audit(
      "{\"op_id\":32,\"params\":[1.5,-0.25],\"signature\":\"scale_add|1.5\",\"template\":\"scale_add\","
      "\"ts_ns\":99,\"version\":16}\n");
  auto recs = OperatorTable::parse_audit_jsonl(audit);
  REQUIRE(recs.size() == 1);
  CHECK(recs[0].op_id == 32);
  CHECK(recs[0].params == (std::vector<double>{1.5, -0.25}));
  CHECK(recs[0].version == 16);
}
