// Builtin operator registry (reference ops.hpp:31-75, 593-623).  The task
// bodies themselves are sm_100a device functions (csrc/ops_*.cuh); this header
// carries the fixed ids, names and limits the host routes by.
#pragma once

#include <cstdint>

#include "gpuos_cuda.h"

namespace gpuos {

enum class OpKind : uint32_t {
  Add = GPUOS_OP_ADD,
  Mul = GPUOS_OP_MUL,
  Relu = GPUOS_OP_RELU,
  Gelu = GPUOS_OP_GELU,
  Softmax = GPUOS_OP_SOFTMAX,
  LayerNorm = GPUOS_OP_LAYERNORM,
  ReduceSum = GPUOS_OP_REDUCE_SUM,
  ReduceMax = GPUOS_OP_REDUCE_MAX,
  ReduceMin = GPUOS_OP_REDUCE_MIN,
  MatMulSmall = GPUOS_OP_MATMUL_SMALL,
  VecMat = GPUOS_OP_VECMAT,
  Sdpa = GPUOS_OP_SDPA,
  Rope = GPUOS_OP_ROPE,
  KvAppend = GPUOS_OP_KV_APPEND,
};

inline constexpr uint32_t kNumBuiltinOps = GPUOS_NUM_BUILTINS;
inline constexpr uint64_t kFirstInjectedId = GPUOS_FIRST_INJECTED_ID;
inline constexpr int64_t kSmallMatmulMaxDim = GPUOS_SMALL_MATMUL_MAX_DIM;

inline const char* op_kind_name(OpKind kind) {
  static constexpr const char* kNames[] = {"add",          "mul",        "relu",       "gelu",   "softmax",
                                           "layernorm",    "reduce_sum", "reduce_max", "reduce_min",
                                           "matmul_small", "vecmat",     "sdpa",       "rope",   "kv_append"};
  const uint32_t i = static_cast<uint32_t>(kind);
  return i < kNumBuiltinOps ? kNames[i] : "unknown";
}

inline bool is_builtin_id(uint64_t op_id) { return op_id < kNumBuiltinOps; }

}  // namespace gpuos
