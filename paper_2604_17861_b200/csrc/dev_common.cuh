// Device-side building blocks shared by every task body: the worker-group
// context, dtype traits that reproduce the reference's load-as-double /
// narrow-once-on-store semantics (reference tensor.hpp:345-371), broadcast
// + dimension coalescing of rank<=4 views (tensor.hpp:190-233), fast divmod
// for strided addressing, and system/gpu-scope memory primitives.
#pragma once

#include "gpuos_cuda.h"  // fixed-width types (NVRTC-safe)
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "gpuos_cuda.h"

namespace gdev {

// ---------------------------------------------------------------------------
// Worker-group context handed to every task body.
// ---------------------------------------------------------------------------
struct Ctx {
  int tid;          // thread index within the worker group
  int nthreads;     // group size (multiple of 32)
  int part;         // partition of the task handled by this group
  int nparts;       // number of partitions the task is split into
  int bar_id;       // named barrier id owned by the group
  int smem_bytes;   // scratch bytes at `smem`
  char* smem;       // shared-memory scratch (no static __shared__ in bodies)
  uint64_t aux;     // table-entry payload (program pointer for KIND_PROGRAM)
  uint32_t flags;   // task flags (GPUOS_FLAG_UNCAPPED, ...)
  uint32_t tmem;    // this group's 128 TMEM columns (kNoTmem = none)
  uint64_t* mbar;   // this group's MMA-completion mbarrier (shared memory)
  uint32_t* mma_phase;  // its current phase bit (shared memory)
};
constexpr uint32_t kNoTmem = 0xffffffffu;

typedef int (*OpFn)(const gpuos_task* t, const Ctx* c);

// Task bodies synchronise their worker group on its own named barrier
// (Ctx::bar_id; barrier 0 is the whole CTA).
__device__ __forceinline__ void group_sync(const Ctx* c) {
  asm volatile("bar.sync %0, %1;" ::"r"(c->bar_id), "r"(c->nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// Memory-model primitives.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sc_sys() { asm volatile("fence.sc.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// 16-byte volatile load of host (mapped pinned) memory; one PCIe read per lane group.
__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
  uint4 v;
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
// Streaming 16-byte load that bypasses L1 (ld.global.cg): a persistent kernel
// never sees a kernel-launch L1 flush, so task inputs written by another SM
// must not be served from this SM's L1.
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Slot checksum term: word i weighted by the odd constant 2i+1 (mod 2^64).
// The host sums it over the 48 words of a slot with word 7 (the checksum)
// left out; the device recomputes the sum warp-wide.  A stale 16-byte chunk
// from the slot's previous lap changes the sum unless its difference is 0,
// so torn reads (queue.hpp:249-251) are caught at ~1 multiply-add per word.
__host__ __device__ __forceinline__ uint64_t slot_term(uint64_t w, uint32_t i) {
  return w * (uint64_t)(2 * i + 1);
}

// ---------------------------------------------------------------------------
// dtype traits.  load() widens to double exactly; narrow() is the single
// rounding a BoundView::store performs (tensor.hpp:354-371).
//
// Coherence rule of the persistent worker: every read of task operand memory
// is an L2 load (gload / load_any / ld_cg_v4: ld.global.cg).  The kernel never
// relaunches, so this SM's L1 may hold lines from earlier tasks that other SMs
// or the host's copy engine have since rewritten; L2 is the coherence point
// (writers release to L2 before their completion is posted).  load() is for
// values already in registers.
// ---------------------------------------------------------------------------
// static_cast<int32_t>(double) on x86 (cvttsd2si): truncation toward zero,
// INT32_MIN for NaN or out of range.  GPU cvt.rzi saturates, so
// the x86 result is reproduced explicitly.
__host__ __device__ __forceinline__ int32_t narrow_i32(double v) {
  if (v > -2147483649.0 && v < 2147483648.0) return (int32_t)v;  // NaN fails both
  return (int32_t)0x80000000u;
}

template <int DT>
struct DT_;
template <>
struct DT_<GPUOS_F32> {
  typedef float T;
  static __device__ __forceinline__ double load(const T* p) { return (double)*p; }
  static __device__ __forceinline__ double gload(const T* p) { return (double)__ldcg(p); }
  static __device__ __forceinline__ void store(T* p, double v) { *p = __double2float_rn(v); }
  static __device__ __forceinline__ double narrow(double v) { return (double)__double2float_rn(v); }
};
template <>
struct DT_<GPUOS_F64> {
  typedef double T;
  static __device__ __forceinline__ double load(const T* p) { return *p; }
  static __device__ __forceinline__ double gload(const T* p) { return __ldcg(p); }
  static __device__ __forceinline__ void store(T* p, double v) { *p = v; }
  static __device__ __forceinline__ double narrow(double v) { return v; }
};
template <>
struct DT_<GPUOS_I32> {
  typedef int32_t T;
  static __device__ __forceinline__ double load(const T* p) { return (double)*p; }
  static __device__ __forceinline__ double gload(const T* p) { return (double)__ldcg(p); }
  static __device__ __forceinline__ void store(T* p, double v) { *p = narrow_i32(v); }
  static __device__ __forceinline__ double narrow(double v) { return (double)narrow_i32(v); }
};
template <>
struct DT_<GPUOS_F16> {
  typedef __half T;
  static __device__ __forceinline__ double load(const T* p) { return (double)__half2float(*p); }
  static __device__ __forceinline__ double gload(const T* p) { return (double)__half2float(__ldcg(p)); }
  static __device__ __forceinline__ void store(T* p, double v) { *p = __double2half(v); }
  static __device__ __forceinline__ double narrow(double v) { return (double)__half2float(__double2half(v)); }
};
template <>
struct DT_<GPUOS_BF16> {
  typedef __nv_bfloat16 T;
  static __device__ __forceinline__ double load(const T* p) { return (double)__bfloat162float(*p); }
  static __device__ __forceinline__ double gload(const T* p) { return (double)__bfloat162float(__ldcg(p)); }
  static __device__ __forceinline__ void store(T* p, double v) { *p = __double2bfloat16(v); }
  static __device__ __forceinline__ double narrow(double v) {
    return (double)__bfloat162float(__double2bfloat16(v));
  }
};

__host__ __device__ __forceinline__ int dtype_width(int dt) {
  return dt == GPUOS_F64 ? 8 : (dt == GPUOS_F16 || dt == GPUOS_BF16) ? 2 : 4;
}

// Runtime-dtype element access (used where per-element cost is dominated by
// math, e.g. rope/sdpa/matmul staging).
__device__ __forceinline__ double load_any(int dt, const char* base, int64_t elem) {
  switch (dt) {
    case GPUOS_F32: return (double)__ldcg((const float*)base + elem);
    case GPUOS_F64: return __ldcg((const double*)base + elem);
    case GPUOS_I32: return (double)__ldcg((const int32_t*)base + elem);
    case GPUOS_F16: return (double)__half2float(__ldcg((const __half*)base + elem));
    default: return (double)__bfloat162float(__ldcg((const __nv_bfloat16*)base + elem));
  }
}
__device__ __forceinline__ void store_any(int dt, char* base, int64_t elem, double v) {
  switch (dt) {
    case GPUOS_F32: ((float*)base)[elem] = __double2float_rn(v); break;
    case GPUOS_F64: ((double*)base)[elem] = v; break;
    case GPUOS_I32: ((int32_t*)base)[elem] = narrow_i32(v); break;
    case GPUOS_F16: ((__half*)base)[elem] = __double2half(v); break;
    default: ((__nv_bfloat16*)base)[elem] = __double2bfloat16(v); break;
  }
}
__device__ __forceinline__ double narrow_any(int dt, double v) {
  switch (dt) {
    case GPUOS_F32: return (double)__double2float_rn(v);
    case GPUOS_F64: return v;
    case GPUOS_I32: return (double)narrow_i32(v);
    case GPUOS_F16: return (double)__half2float(__double2half(v));
    default: return (double)__bfloat162float(__double2bfloat16(v));
  }
}

// ---------------------------------------------------------------------------
// View checks that mirror the reference helpers (ops.hpp:84-128).
// ---------------------------------------------------------------------------
// BoundView construction (tensor.hpp:337-343): unknown buffer, dtype vs buffer.
__device__ __forceinline__ int bind_code(const gpuos_view& v) {
  switch (v.status) {
    case GPUOS_VIEW_OK: return GPUOS_OK;
    case GPUOS_VIEW_UNKNOWN_BUFFER: return GPUOS_INVALID_BUFFER;
    case GPUOS_VIEW_DTYPE_VS_BUFFER: return GPUOS_DTYPE_MISMATCH;
    default: return GPUOS_OUT_OF_BOUNDS;
  }
}
__device__ __forceinline__ int64_t numel(const gpuos_view& v) {
  int64_t n = 1;
  for (int d = 0; d < v.rank; ++d) n *= v.extents[d];
  return n;
}
__device__ __forceinline__ bool same_shape(const gpuos_view& a, const gpuos_view& b) {
  if (a.rank != b.rank) return false;
  for (int d = 0; d < a.rank; ++d)
    if (a.extents[d] != b.extents[d]) return false;
  return true;
}
__device__ __forceinline__ bool is_float_dt(int dt) { return dt != GPUOS_I32; }
// Row-major contiguous (unit dims ignored): element e lives at offset e.
__device__ __forceinline__ bool dense_view(const gpuos_view& v) {
  int64_t expect = 1;
  for (int d = v.rank - 1; d >= 0; --d) {
    if (v.extents[d] == 1) continue;
    if (v.strides[d] != expect) return false;
    expect *= v.extents[d];
  }
  return true;
}

// ---------------------------------------------------------------------------
// Task plan: a shape classification computed once per task before the body
// runs (by the fetcher warp in the worker, by the kernel prologue on the
// conventional path) and handed over in Ctx::flags.  kPlanDenseSame means
// every operand view (output + n_inputs inputs) bound cleanly, has the
// output's dtype and shape, and is row-major dense: every reference check an
// elementwise body performs would pass, so it may go straight to its dense
// loop.  The plan is only a hint; bodies must still be correct without it.
// ---------------------------------------------------------------------------
constexpr uint32_t kPlanDenseSame = 1u << 31;

// View `k`'s part of the classification (one lane per view).
__device__ __forceinline__ bool plan_view_ok(const gpuos_task* t, int k) {
  const gpuos_view& o = t->views[0];
  const gpuos_view& v = t->views[k];
  return v.status == GPUOS_VIEW_OK && v.dtype == o.dtype && same_shape(v, o) && dense_view(v);
}
// Warp-wide classification: lanes 0..n_inputs each check one view.
__device__ __forceinline__ uint32_t plan_task_warp(const gpuos_task* t, int lane) {
  const int nv = 1 + (int)t->n_inputs;
  const bool ok = lane >= nv || nv > 1 + GPUOS_MAX_INPUTS || plan_view_ok(t, lane);
  const unsigned all = __all_sync(0xffffffffu, ok);
  return (all && nv <= 1 + GPUOS_MAX_INPUTS) ? kPlanDenseSame : 0u;
}

// ---------------------------------------------------------------------------
// Fast unsigned divmod by an invariant divisor (n < 2^31).
// ---------------------------------------------------------------------------
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ void init(uint32_t div) {
    d = div;
    s = 0;
    while ((1u << s) < div) ++s;
    m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

// ---------------------------------------------------------------------------
// Multi-operand strided iteration space: up to 5 operands (out + 4 inputs)
// broadcast to the output shape, unit dims dropped, mergeable dims coalesced.
// ---------------------------------------------------------------------------
struct Space {
  int rank;                  // coalesced rank (0 => single element)
  int nops;                  // operands (0 = output)
  int32_t ext[GPUOS_MAX_RANK];
  int64_t st[5][GPUOS_MAX_RANK];  // element strides per operand
  FastDiv fd[GPUOS_MAX_RANK];
  bool dense;                // every operand is contiguous with the output's layout
};

// Right-aligned broadcast of `in` to `out`'s shape (tensor.hpp:208-233):
// writes per-out-dim strides; returns false on IncompatibleShapes.
__device__ __forceinline__ bool broadcast_strides(const gpuos_view& in, const gpuos_view& out,
                                                  int64_t* st) {
  const int ro = out.rank, ri = in.rank;
  if (ri > ro) return false;
  for (int d = 0; d < ro; ++d) st[d] = 0;
  for (int i = 0; i < ri; ++i) {
    const int dv = in.extents[ri - 1 - i], dt = out.extents[ro - 1 - i];
    if (dv == dt) {
      st[ro - 1 - i] = in.strides[ri - 1 - i];
    } else if (dv == 1) {
      st[ro - 1 - i] = 0;
    } else {
      return false;
    }
  }
  return true;
}

// Build the iteration space from the output view and per-operand strides
// aligned to the output dims (st_in[k][d] for operand k+1).
__device__ __forceinline__ void build_space(Space& s, const gpuos_view& out, int n_in,
                                            const int64_t (*st_in)[GPUOS_MAX_RANK]) {
  s.nops = n_in + 1;
  // drop unit dims
  int r = 0;
  int32_t ext[GPUOS_MAX_RANK];
  int64_t st[5][GPUOS_MAX_RANK];
  for (int d = 0; d < out.rank; ++d) {
    if (out.extents[d] == 1) continue;
    ext[r] = out.extents[d];
    st[0][r] = out.strides[d];
    for (int k = 0; k < n_in; ++k) st[k + 1][r] = st_in[k][d];
    ++r;
  }
  // coalesce: merge dim d into d+1 when stride[d] == stride[d+1]*ext[d+1] for all operands
  int w = 0;
  for (int d = 0; d < r; ++d) {
    if (w > 0) {
      bool ok = true;
      for (int k = 0; k <= n_in; ++k)
        if (st[k][w - 1] != st[k][d] * (int64_t)ext[d]) ok = false;
      if (ok) {
        ext[w - 1] *= ext[d];
        for (int k = 0; k <= n_in; ++k) st[k][w - 1] = st[k][d];
        continue;
      }
    }
    ext[w] = ext[d];
    for (int k = 0; k <= n_in; ++k) st[k][w] = st[k][d];
    ++w;
  }
  s.rank = w;
  bool dense = (w <= 1);
  for (int k = 0; k <= n_in && dense; ++k)
    if (w == 1 && st[k][0] != 1) dense = false;
  s.dense = dense;
  for (int d = 0; d < w; ++d) {
    s.ext[d] = ext[d];
    s.fd[d].init((uint32_t)ext[d]);
    for (int k = 0; k <= n_in; ++k) s.st[k][d] = st[k][d];
  }
}

// Element offsets of linear index e (row-major over the coalesced space).
__device__ __forceinline__ void space_offsets(const Space& s, uint32_t e, int64_t* off) {
  for (int k = 0; k < s.nops; ++k) off[k] = 0;
  for (int d = s.rank - 1; d >= 0; --d) {
    const uint32_t q = s.fd[d].div(e);
    const uint32_t i = e - q * s.fd[d].d;
    e = q;
    for (int k = 0; k < s.nops; ++k) off[k] += (int64_t)i * s.st[k][d];
  }
}

// Partition [0, n) into nparts chunks aligned to `align` elements.
__device__ __forceinline__ void part_range(int64_t n, int part, int nparts, int64_t align,
                                           int64_t* lo, int64_t* hi) {
  if (nparts <= 1) {
    *lo = 0;
    *hi = n;
    return;
  }
  int64_t chunk = (n + nparts - 1) / nparts;
  chunk = (chunk + align - 1) / align * align;
  int64_t a = (int64_t)part * chunk, b = a + chunk;
  if (a > n) a = n;
  if (b > n) b = n;
  *lo = a;
  *hi = b;
}

// ---------------------------------------------------------------------------
// Group reductions (warp shuffle + shared-memory staging).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = v < x ? x : v;
  }
  return v;
}
// Sum over the whole group; every thread gets the result.  `red` must hold
// nthreads/32 doubles of scratch; the call contains two group barriers.
__device__ __forceinline__ double group_sum(double v, const Ctx* c, double* red) {
  v = warp_sum(v);
  const int lane = c->tid & 31, wid = c->tid >> 5, nw = c->nthreads >> 5;
  if (lane == 0) red[wid] = v;
  group_sync(c);
  double t = 0.0;
  for (int i = 0; i < nw; ++i) t += red[i];
  group_sync(c);
  return t;
}
__device__ __forceinline__ double group_max(double v, const Ctx* c, double* red) {
  v = warp_max(v);
  const int lane = c->tid & 31, wid = c->tid >> 5, nw = c->nthreads >> 5;
  if (lane == 0) red[wid] = v;
  group_sync(c);
  double t = red[0];
  for (int i = 1; i < nw; ++i) t = t < red[i] ? red[i] : t;
  group_sync(c);
  return t;
}

}  // namespace gdev
