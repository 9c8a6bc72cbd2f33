/*
 * gpuos_oracle.h — CPU restatement of the reference task bodies (TEST
 * INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  It restates, in plain C over
 * raw buffers, the arithmetic of /root/reference/proj/include/gpuos/ops.hpp,
 * tensor.hpp, expr.hpp and bytecode.hpp; every function cites the lines it
 * follows.  F32/F64/I32 parity is pinned against the reference itself
 * (oracle/_ref/libref.so and tests/golden/); F16/BF16 are new dtypes the
 * reference does not have, so their narrowing (round-to-nearest-even from
 * the exact double, tensor.hpp:354-371's single-rounding rule) is a labelled
 * restatement — parity unpinned for those two dtypes.
 */
#ifndef GPUOS_ORACLE_H_
#define GPUOS_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_RANK 8

/* dtype codes follow include/gpuos_cuda.h */
enum { ORC_F32 = 0, ORC_F64 = 1, ORC_I32 = 2, ORC_F16 = 3, ORC_BF16 = 4 };

/* A TensorView (tensor.hpp:66-94) bound to its buffer (BoundView). */
typedef struct orc_view {
  void* base;         /* buffer element 0 */
  int64_t offset;     /* elements */
  int32_t rank;
  int32_t dtype;      /* view dtype */
  int64_t shape[ORC_MAX_RANK];
  int64_t strides[ORC_MAX_RANK];
  int32_t buf_dtype;  /* dtype of the owning buffer; -1 = unknown buffer */
  int32_t pad;
} orc_view;

/* Conversions (tensor.hpp:259-285 plus the F16/BF16 restatement). */
double orc_load(int dtype, const void* base, int64_t elem);
void orc_store(int dtype, void* base, int64_t elem, double v);
double orc_narrow(int dtype, double v);
uint16_t orc_f16_bits(double v);
uint16_t orc_bf16_bits(double v);
double orc_f16_value(uint16_t b);
double orc_bf16_value(uint16_t b);
int32_t orc_narrow_i32(double v);

/* Builtin bodies; return the reference ErrorCode (0 = Ok). */
int orc_elementwise(int op, orc_view* out, orc_view* inputs, int n_inputs); /* 0 add 1 mul 2 relu 3 gelu */
int orc_softmax(orc_view* out, orc_view* in);
int orc_layernorm(orc_view* out, orc_view* in, orc_view* gamma, orc_view* beta, double eps, int has_eps);
int orc_reduce(int mode, orc_view* out, orc_view* in); /* 0 sum 1 max 2 min */
int orc_matmul(orc_view* out, orc_view* a, orc_view* b, int64_t max_dim);
int orc_vecmat(orc_view* out, orc_view* v, orc_view* m, int64_t max_dim);
int orc_sdpa(orc_view* out, orc_view* q, orc_view* k, orc_view* v, double scale_override, int has_scale);
int orc_rope(orc_view* out, orc_view* x, orc_view* pos, double base_override, int has_base);
int orc_kv_append(orc_view* k_cache, orc_view* v_cache, orc_view* new_k, orc_view* new_v, double cursor);

/* Injected operators: stack-machine program (bytecode.hpp:205-230) evaluated
 * over broadcast inputs (opcompiler.hpp:70-122).  code = n x {op, k, value}. */
typedef struct orc_instr {
  int32_t op;
  int32_t k;
  double value;
} orc_instr;
int orc_program(const orc_instr* code, int n, int arity, int dtype, orc_view* out, orc_view* inputs, int n_inputs);

/* Broadcast helpers (tensor.hpp:104-147); return 0 or IncompatibleShapes. */
int orc_broadcast_shapes(const int64_t* a, int ra, const int64_t* b, int rb, int64_t* out, int* rout);

#ifdef __cplusplus
}
#endif
#endif
