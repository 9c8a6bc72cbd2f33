// ref_shim.cpp — TEST INFRASTRUCTURE: exposes the unmodified reference task
// bodies (compiled from /root/reference/proj/include, never copied) through
// a C ABI so tests/ can pin oracle/gpuos_oracle.c against the reference
// itself.  Built into oracle/_ref/libref.so by oracle/Makefile.
#include <gpuos/ops.hpp>
#include <gpuos/opcompiler.hpp>

#include <cstring>
#include <vector>

using namespace gpuos;

extern "C" {

struct ref_tensor {
  void* data;       // host buffer, buf_len elements of dtype
  int64_t buf_len;
  int32_t dtype;    // 0 f32, 1 f64, 2 i32
  int32_t rank;
  int64_t offset;
  int64_t shape[8];
  int64_t strides[8];
};

static TensorView bind_tensor(BufferPool& pool, const ref_tensor& t) {
  TensorView v;
  v.dtype = static_cast<DType>(t.dtype);
  v.buffer = pool.allocate(v.dtype, static_cast<size_t>(t.buf_len));
  std::memcpy(pool.raw(v.buffer), t.data, static_cast<size_t>(t.buf_len) * dtype_width(v.dtype));
  v.offset = t.offset;
  v.shape.assign(t.shape, t.shape + t.rank);
  v.strides.assign(t.strides, t.strides + t.rank);
  return v;
}

// Run builtin `kind` (ops.hpp:31-48) on copies of the tensors; results are
// copied back into every tensor's host buffer.  max_dim <= 0 runs matmul /
// vecmat uncapped (the inline path).  Returns the reference ErrorCode.
int ref_run_builtin(int kind, int n_in, ref_tensor* ins, ref_tensor* out, const double* scalars, int n_sc,
                    int64_t max_dim) {
  BufferPool pool;
  std::vector<TensorView> views;
  for (int i = 0; i < n_in; ++i) views.push_back(bind_tensor(pool, ins[i]));
  TensorView ov = bind_tensor(pool, *out);
  OpContext ctx;
  ctx.pool = &pool;
  ctx.inputs = std::span<const TensorView>(views.data(), views.size());
  ctx.output = &ov;
  ctx.scalars = std::span<const double>(scalars, static_cast<size_t>(n_sc));
  ctx.size = static_cast<uint64_t>(ov.numel());
  int code = 0;
  try {
    const OpKind k = static_cast<OpKind>(kind);
    if (k == OpKind::MatMulSmall && max_dim <= 0) matmul(ctx, 0);
    else if (k == OpKind::VecMat && max_dim <= 0) vecmat(ctx, 0);
    else builtin_fn(k)(ctx);
  } catch (const Error& e) {
    code = static_cast<int>(e.code());
  } catch (...) {
    code = static_cast<int>(ErrorCode::Internal);
  }
  for (int i = 0; i < n_in; ++i)
    std::memcpy(ins[i].data, pool.raw(views[static_cast<size_t>(i)].buffer),
                static_cast<size_t>(ins[i].buf_len) * dtype_width(views[static_cast<size_t>(i)].dtype));
  std::memcpy(out->data, pool.raw(ov.buffer), static_cast<size_t>(out->buf_len) * dtype_width(ov.dtype));
  return code;
}

// Compile a template through the reference ModuleCache and run the loaded
// module (opcompiler.hpp:70-122) — the parity source for injected operators.
int ref_run_template(const char* source, int arity, const double* params, int n_params, int dtype, int n_in,
                     ref_tensor* ins, ref_tensor* out) {
  BufferPool pool;
  std::vector<TensorView> views;
  for (int i = 0; i < n_in; ++i) views.push_back(bind_tensor(pool, ins[i]));
  TensorView ov = bind_tensor(pool, *out);
  int code = 0;
  try {
    ModuleCache cache;
    OperatorTemplate t{"shim", source, arity};
    ModulePtr m = cache.compile_or_get(t, std::span<const double>(params, static_cast<size_t>(n_params)),
                                       static_cast<DType>(dtype));
    OpFn fn = load_module(m);
    OpContext ctx;
    ctx.pool = &pool;
    ctx.inputs = std::span<const TensorView>(views.data(), views.size());
    ctx.output = &ov;
    ctx.size = static_cast<uint64_t>(ov.numel());
    fn(ctx);
  } catch (const Error& e) {
    code = static_cast<int>(e.code());
  } catch (...) {
    code = static_cast<int>(ErrorCode::Internal);
  }
  std::memcpy(out->data, pool.raw(ov.buffer), static_cast<size_t>(out->buf_len) * dtype_width(ov.dtype));
  return code;
}

// Lower + verify through the reference (bytecode.hpp:135-201); writes up to
// cap instructions {op, k, value} and returns the count, or -code on error.
int ref_compile_template(const char* source, const double* params, int n_params, int arity, int32_t* ops,
                         int32_t* ks, double* values, int cap, int* max_stack) {
  try {
    ExprPtr ast = parse_expression(source);
    ExprPtr folded = substitute_params(*ast, std::span<const double>(params, static_cast<size_t>(n_params)));
    Bytecode code = lower(*folded, {});
    *max_stack = verify(code, arity);
    if (static_cast<int>(code.size()) > cap) return -static_cast<int>(ErrorCode::TooLarge);
    for (size_t i = 0; i < code.size(); ++i) {
      ops[i] = static_cast<int32_t>(code[i].op);
      ks[i] = code[i].k;
      values[i] = code[i].value;
    }
    return static_cast<int>(code.size());
  } catch (const Error& e) {
    return -static_cast<int>(e.code());
  }
}

}  // extern "C"
