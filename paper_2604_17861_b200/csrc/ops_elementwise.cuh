// Elementwise task bodies: add / mul / relu / gelu (reference ops.hpp:133-194),
// the injected-operator stack machine (bytecode.hpp:205-230 evaluated by
// opcompiler.hpp:70-122's broadcast driver) and kv_append (ops.hpp:544-589).
//
// Every body evaluates in double and narrows once on store, like the
// reference's BoundView path, so f32/f16/bf16/i32 add/mul/relu are bit-exact.
// The dense path moves 16 bytes per operand per thread with four independent
// vectors in flight; the strided/broadcast path walks a coalesced rank<=4
// space with fast divmod.
#pragma once

#include "dev_common.cuh"
#include "dev_state.h"

namespace gdev {

// ---- scalar functions in reference evaluation order (no contraction) ----
// `f32` is the same function on f32 operands without the round trip through
// double.  It is bit-identical to narrow(op(double(a), double(b))): for + and
// * a double (53-bit) intermediate rounded to f32 (24-bit) is the correctly
// rounded f32 result, since 53 >= 2*24 + 2 (double rounding is innocuous),
// and relu only selects.  No FTZ: nvcc keeps f32 denormals by default.
struct FAdd {
  static constexpr int A = 2;
  static constexpr bool kF32 = true;
  __device__ __forceinline__ double operator()(const double* v) const { return __dadd_rn(v[0], v[1]); }
  __device__ __forceinline__ float f32(const float* v) const { return __fadd_rn(v[0], v[1]); }
  __device__ __forceinline__ long long i64(const long long* v) const { return v[0] + v[1]; }
};
struct FMul {
  static constexpr int A = 2;
  static constexpr bool kF32 = true;
  __device__ __forceinline__ double operator()(const double* v) const { return __dmul_rn(v[0], v[1]); }
  __device__ __forceinline__ float f32(const float* v) const { return __fmul_rn(v[0], v[1]); }
  __device__ __forceinline__ long long i64(const long long* v) const { return v[0] * v[1]; }
};
struct FRelu {
  static constexpr int A = 1;
  static constexpr bool kF32 = true;
  // v < 0 ? 0 : v keeps -0.0 and NaN (ops.hpp:188)
  __device__ __forceinline__ double operator()(const double* v) const { return v[0] < 0.0 ? 0.0 : v[0]; }
  __device__ __forceinline__ float f32(const float* v) const { return v[0] < 0.0f ? 0.0f : v[0]; }
  __device__ __forceinline__ long long i64(const long long* v) const { return v[0] < 0 ? 0 : v[0]; }
};
template <class F, class = void>
struct HasF32 {
  static constexpr bool value = false;
};
template <class F>
struct HasF32<F, decltype((void)F::kF32)> {
  static constexpr bool value = F::kF32;
};
// f32 evaluation of add/mul/relu for the 16- and 32-bit float dtypes.  For
// F16/BF16 the operands widen to f32 exactly, f32 add/mul round once to 24
// bits, and the narrowing to 11 (f16) or 8 (bf16) bits is then the correctly
// rounded result of the exact sum/product -- double rounding is innocuous
// when 24 >= 2q + 2 (q = 11 or 8), the same argument as double -> f32 above;
// f32 subnormals and overflow map to the 16-bit format's the same way.  So
// this is bit-identical to the reference's double evaluation narrowed once.
template <int DT>
struct F32Eval {
  static constexpr bool value = DT == GPUOS_F32 || DT == GPUOS_F16 || DT == GPUOS_BF16;
};
// I32 add/mul/relu in int64: |a + b| < 2^32 and |a * b| < 2^62 are exact,
// and the reference's double result, when it fits int32, is that exact value
// (an out-of-range double narrows to INT32_MIN, as the int64 check does).
template <bool I, class A, class B>
struct PickT {
  typedef A type;
};
template <class A, class B>
struct PickT<false, A, B> {
  typedef B type;
};
template <int DT>
struct FastEval {  // (no <type_traits>: NVRTC compiles this header for native injected ops)
  static constexpr bool value = F32Eval<DT>::value || DT == GPUOS_I32;
  typedef typename PickT<DT == GPUOS_I32, long long, float>::type CT;
};
template <int DT>
__device__ __forceinline__ typename FastEval<DT>::CT to_ct(typename DT_<DT>::T v) {
  if constexpr (DT == GPUOS_I32) return (long long)v;
  else if constexpr (DT == GPUOS_F16) return __half2float(v);
  else if constexpr (DT == GPUOS_BF16) return __bfloat162float(v);
  else return (float)v;
}
template <int DT>
__device__ __forceinline__ typename DT_<DT>::T from_ct(typename FastEval<DT>::CT v) {
  if constexpr (DT == GPUOS_I32) return (v >= -2147483648LL && v <= 2147483647LL) ? (int32_t)v : (int32_t)0x80000000u;
  else if constexpr (DT == GPUOS_F16) return __float2half_rn(v);
  else if constexpr (DT == GPUOS_BF16) return __float2bfloat16_rn(v);
  else return v;
}
template <int DT, class F>
__device__ __forceinline__ typename FastEval<DT>::CT fast_eval(const F& f, const typename FastEval<DT>::CT* x) {
  if constexpr (DT == GPUOS_I32) return f.i64(x);
  else return f.f32(x);
}
template <int DT>
__device__ __forceinline__ float to_f32(typename DT_<DT>::T v) {
  if constexpr (DT == GPUOS_F16) return __half2float(v);
  else if constexpr (DT == GPUOS_BF16) return __bfloat162float(v);
  else return (float)v;
}
template <int DT>
__device__ __forceinline__ typename DT_<DT>::T from_f32(float v) {
  if constexpr (DT == GPUOS_F16) return __float2half_rn(v);
  else if constexpr (DT == GPUOS_BF16) return __float2bfloat16_rn(v);
  else return v;
}

struct FGelu {
  static constexpr int A = 1;
  // 0.5 * x * (1 + tanh(c * (x + 0.044715 * x * x * x))), c = sqrt(2/pi)  (ops.hpp:79-82)
  __device__ __forceinline__ double operator()(const double* v) const {
    const double x = v[0];
    const double c = 0x1.9884533d43651p-1;  // sqrt(2.0 / pi) as glibc computes it
    const double x3 = __dmul_rn(__dmul_rn(__dmul_rn(0.044715, x), x), x);
    const double inner = __dmul_rn(c, __dadd_rn(x, x3));
    return __dmul_rn(__dmul_rn(0.5, x), __dadd_rn(1.0, tanh(inner)));
  }
};

// ---- the shared elementwise driver ----
// kAligned: the caller has checked every operand is 16-byte aligned, so the
// element-wise (unaligned) loop is not instantiated -- the worker's inline
// path uses this to stay within its register budget.
template <int DT, class F, int U = 4, bool kAligned = false>
__device__ __forceinline__ void ew_dense(const gpuos_task* t, const Ctx* c, int64_t n, F f) {
  typedef typename DT_<DT>::T T;
  constexpr int A = F::A;
  T* out = (T*)t->views[0].addr;
  const T* in[A];
#pragma unroll
  for (int k = 0; k < A; ++k) in[k] = (const T*)t->views[1 + k].addr;
  bool aligned = ((uintptr_t)out & 15) == 0;
#pragma unroll
  for (int k = 0; k < A; ++k) aligned = aligned && (((uintptr_t)in[k] & 15) == 0);
  constexpr int V = 16 / sizeof(T);
  int64_t tail_lo = 0;
  if (kAligned || aligned) {
    const int64_t nv = n / V;
    int64_t lo, hi;
    part_range(nv, c->part, c->nparts, 1, &lo, &hi);
    const int stride = c->nthreads;
    for (int64_t i0 = lo + c->tid; i0 < hi; i0 += (int64_t)stride * U) {
      uint4 vin[A][U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + (int64_t)u * stride;
        if (i < hi) {
#pragma unroll
          for (int k = 0; k < A; ++k) vin[k][u] = ld_cg_v4(reinterpret_cast<const uint4*>(in[k]) + i);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + (int64_t)u * stride;
        if (i < hi) {
          uint4 vo;
          const T* ev[A];
#pragma unroll
          for (int k = 0; k < A; ++k) ev[k] = reinterpret_cast<const T*>(&vin[k][u]);
          T* eo = reinterpret_cast<T*>(&vo);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            if constexpr (FastEval<DT>::value && HasF32<F>::value) {
              typename FastEval<DT>::CT x[A];
#pragma unroll
              for (int k = 0; k < A; ++k) x[k] = to_ct<DT>(ev[k][j]);
              eo[j] = from_ct<DT>(fast_eval<DT>(f, x));
            } else {
              double x[A];
#pragma unroll
              for (int k = 0; k < A; ++k) x[k] = DT_<DT>::load(ev[k] + j);
              DT_<DT>::store(eo + j, f(x));
            }
          }
          reinterpret_cast<uint4*>(out)[i] = vo;
        }
      }
    }
    if (c->part != c->nparts - 1) return;  // the last partition owns the scalar tail
    tail_lo = nv * V;
  } else if constexpr (!kAligned) {
    // an operand is not 16-byte aligned (views at arbitrary element offsets):
    // element loads, still coalesced across the warp, with UE elements per
    // thread in flight so a round costs one memory latency, not UE.  f32
    // add/mul/relu stay in f32 registers (bit-identical, see FAdd), which
    // halves the registers per element in flight.  (A funnel-shifted 16-byte
    // vector variant -- two aligned blocks per vector, or one block plus a
    // lane shuffle -- measured slower here: 7.6-8.0M vs 13.8M config-2 tasks/s.)
    int64_t lo, hi;
    part_range(n, c->part, c->nparts, 1, &lo, &hi);
    if constexpr (FastEval<DT>::value && HasF32<F>::value) {
      typedef typename FastEval<DT>::CT CT;
      constexpr int UE = 16;
      const int64_t step = (int64_t)c->nthreads * UE;
      for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
        CT x[UE][A];
#pragma unroll
        for (int u = 0; u < UE; ++u) {
          const int64_t e = e0 + (int64_t)u * c->nthreads;
          if (e < hi) {
#pragma unroll
            for (int k = 0; k < A; ++k) x[u][k] = to_ct<DT>(__ldcg(in[k] + e));
          }
        }
#pragma unroll
        for (int u = 0; u < UE; ++u) {
          const int64_t e = e0 + (int64_t)u * c->nthreads;
          if (e < hi) out[e] = from_ct<DT>(fast_eval<DT>(f, x[u]));
        }
      }
      return;
    }
    constexpr int UE = 8;
    const int64_t step = (int64_t)c->nthreads * UE;
    for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
      double x[UE][A];
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) {
#pragma unroll
          for (int k = 0; k < A; ++k) x[u][k] = DT_<DT>::gload(in[k] + e);
        }
      }
#pragma unroll
      for (int u = 0; u < UE; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) DT_<DT>::store(out + e, f(x[u]));
      }
    }
    return;
  }
  for (int64_t e = tail_lo + c->tid; e < n; e += c->nthreads) {
    double x[A];
#pragma unroll
    for (int k = 0; k < A; ++k) x[k] = DT_<DT>::gload(in[k] + e);
    DT_<DT>::store(out + e, f(x));
  }
}

// One coalesced dimension with per-operand element strides st[0..A] (st[0]
// the output's): stride-k views, rank-0 scalars, row-major views of any rank
// that flatten to a single stride.  Offsets are e * stride; no divmod.
template <int DT, class F>
__device__ __forceinline__ void ew_rank1(const gpuos_task* t, const Ctx* c, int64_t n, F f, const int64_t* stp) {
  typedef typename DT_<DT>::T T;
  constexpr int A = F::A;
  int64_t st[1 + A];  // in registers: through the pointer, every output store would force a reload
#pragma unroll
  for (int k = 0; k <= A; ++k) st[k] = stp[k];
  T* out = (T*)t->views[0].addr;
  const T* in[A];
#pragma unroll
  for (int k = 0; k < A; ++k) in[k] = (const T*)t->views[1 + k].addr;
  int64_t lo, hi;
  part_range(n, c->part, c->nparts, 1, &lo, &hi);
  if constexpr (FastEval<DT>::value && HasF32<F>::value) {
    typedef typename FastEval<DT>::CT CT;
    constexpr int U1F = 16;
    const int64_t stepf = (int64_t)c->nthreads * U1F;
    for (int64_t e0 = lo + c->tid; e0 < hi; e0 += stepf) {
      CT x[U1F][A];
#pragma unroll
      for (int u = 0; u < U1F; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) {
#pragma unroll
          for (int k = 0; k < A; ++k) x[u][k] = to_ct<DT>(__ldcg(in[k] + e * st[1 + k]));
        }
      }
#pragma unroll
      for (int u = 0; u < U1F; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) out[e * st[0]] = from_ct<DT>(fast_eval<DT>(f, x[u]));
      }
    }
  } else {
    constexpr int U1 = 8;
    const int64_t step = (int64_t)c->nthreads * U1;
    for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
      double x[U1][A];
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) {
#pragma unroll
          for (int k = 0; k < A; ++k) x[u][k] = DT_<DT>::gload(in[k] + e * st[1 + k]);
        }
      }
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) DT_<DT>::store(out + e * st[0], f(x[u]));
      }
    }
  }
}

// Register-resident broadcast check: the element stride of `in` against a
// row-major dense output of the same rank-aligned shape when the view
// flattens to one stride (every non-unit output dim d: stride_d == s *
// out_stride_d), with s = 0 for a broadcast scalar.  Fixed-bound loops keep
// everything in registers; the general Space build indexes small arrays at
// run time, which lands in local memory -- measured 16,000 cycles of setup
// for a 2,048-element broadcast half-task vs 2,000 for a dense one.
__device__ __forceinline__ bool flat_stride(const gpuos_view& in, const gpuos_view& out, int64_t* s) {
  const int ro = out.rank, ri = in.rank;
  if (ri > ro) return false;
  int64_t st = 0;
  bool have = false, ok = true;
#pragma unroll
  for (int d = GPUOS_MAX_RANK - 1; d >= 0; --d) {
    if (d < ro) {
      const int di = d - (ro - ri);  // the input dim aligned with output dim d (right-aligned)
      const int32_t eo = out.extents[d];
      int32_t ei = 1, si = 0;
#pragma unroll
      for (int q = 0; q < GPUOS_MAX_RANK; ++q)
        if (q == di) {
          ei = in.extents[q];
          si = in.strides[q];
        }
      if (di >= 0 && ei != eo && ei != 1) ok = false;  // incompatible: let the general path report it
      const int64_t sd = (di >= 0 && ei == eo) ? si : 0;  // broadcast dims read stride 0
      if (eo != 1) {
        if (!have) {
          // innermost non-unit dim: out stride there is the unit of the flat index
          if (sd % out.strides[d] != 0) ok = false;
          st = sd / out.strides[d];
          have = true;
        } else if (sd != st * out.strides[d]) {
          ok = false;
        }
      }
    }
  }
  *s = st;
  return ok;
}

template <int DT, class F>
__device__ __forceinline__ void ew_strided(const gpuos_task* t, const Ctx* c, const Space& s,
                                           int64_t n, F f) {
  typedef typename DT_<DT>::T T;
  constexpr int A = F::A;
  T* out = (T*)t->views[0].addr;
  const T* in[A];
#pragma unroll
  for (int k = 0; k < A; ++k) in[k] = (const T*)t->views[1 + k].addr;
  int64_t lo, hi;
  part_range(n, c->part, c->nparts, 1, &lo, &hi);
  if (s.rank == 1) {
    // one coalesced dimension (stride-k views, rank-0 / row broadcasts over a
    // flat output): offsets are e * stride, no divmod, strides in registers
    int64_t st[1 + A];
#pragma unroll
    for (int k = 0; k <= A; ++k) st[k] = s.st[k][0];
    if constexpr (FastEval<DT>::value && HasF32<F>::value) {
      typedef typename FastEval<DT>::CT CT;
      constexpr int U1F = 16;
      const int64_t stepf = (int64_t)c->nthreads * U1F;
      for (int64_t e0 = lo + c->tid; e0 < hi; e0 += stepf) {
        CT x[U1F][A];
#pragma unroll
        for (int u = 0; u < U1F; ++u) {
          const int64_t e = e0 + (int64_t)u * c->nthreads;
          if (e < hi) {
#pragma unroll
            for (int k = 0; k < A; ++k) x[u][k] = to_ct<DT>(__ldcg(in[k] + e * st[1 + k]));
          }
        }
#pragma unroll
        for (int u = 0; u < U1F; ++u) {
          const int64_t e = e0 + (int64_t)u * c->nthreads;
          if (e < hi) out[e * st[0]] = from_ct<DT>(fast_eval<DT>(f, x[u]));
        }
      }
      return;
    }
    constexpr int U1 = 8;
    const int64_t step = (int64_t)c->nthreads * U1;
    for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
      double x[U1][A];
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) {
#pragma unroll
          for (int k = 0; k < A; ++k) x[u][k] = DT_<DT>::gload(in[k] + e * st[1 + k]);
        }
      }
#pragma unroll
      for (int u = 0; u < U1; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) DT_<DT>::store(out + e * st[0], f(x[u]));
      }
    }
    return;
  }
  if (s.rank == 2) {
    // two coalesced dims (row broadcasts, transposed 2-D views): strides and
    // the column divisor in registers, one divmod per element
    int64_t st0[1 + A], st1[1 + A];
#pragma unroll
    for (int k = 0; k <= A; ++k) {
      st0[k] = s.st[k][0];
      st1[k] = s.st[k][1];
    }
    const FastDiv fd = s.fd[1];
    if constexpr (FastEval<DT>::value && HasF32<F>::value) {
      typedef typename FastEval<DT>::CT CT;
      // 32-bit offsets when every operand's span fits (config-2 views do)
      int64_t span = 0;
#pragma unroll
      for (int k = 0; k <= A; ++k) {
        const int64_t a0 = st0[k] < 0 ? -st0[k] : st0[k], a1 = st1[k] < 0 ? -st1[k] : st1[k];
        const int64_t sp = a0 * (s.ext[0] - 1) + a1 * (s.ext[1] - 1);
        span = sp > span ? sp : span;
      }
      if (span < ((int64_t)1 << 31)) {
        int32_t s0[1 + A], s1[1 + A];
#pragma unroll
        for (int k = 0; k <= A; ++k) {
          s0[k] = (int32_t)st0[k];
          s1[k] = (int32_t)st1[k];
        }
        // Transposed inputs (row stride 1, column stride > 1) against a
        // row-major output: 32x32 tiles per warp through shared memory, so
        // both the column-major reads and the row-major writes coalesce.
        bool tr[A];
        bool any_tr = false;
#pragma unroll
        for (int k = 0; k < A; ++k) {
          tr[k] = s0[1 + k] == 1 && (s1[1 + k] > 1 || s1[1 + k] < -1);
          any_tr = any_tr || tr[k];
        }
        const int nw = c->nthreads >> 5;
        if (any_tr && s1[0] == 1 && c->smem_bytes >= nw * A * 32 * 33 * 4 && s.ext[0] >= 8) {
          const int lane = c->tid & 31, warp = c->tid >> 5;
          const int R = s.ext[0], C = s.ext[1];
          const int tcols = (C + 31) / 32;
          const int64_t ntiles = (int64_t)((R + 31) / 32) * tcols;
          int64_t tlo, thi;
          part_range(ntiles, c->part, c->nparts, 1, &tlo, &thi);
          T* tile = reinterpret_cast<T*>(c->smem) + (size_t)warp * A * 32 * 33;  // raw elements
          for (int64_t tt = tlo + warp; tt < thi; tt += nw) {
            const int q0 = (int)(tt / tcols) * 32, r0 = (int)(tt % tcols) * 32;
#pragma unroll
            for (int k = 0; k < A; ++k) {
              if (!tr[k]) continue;
              T v[32];
              const int q = q0 + lane;
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (q < R && r0 + i < C) v[i] = __ldcg(in[k] + (q * s0[1 + k] + (r0 + i) * s1[1 + k]));
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (q < R && r0 + i < C) tile[(k * 32 + i) * 33 + lane] = v[i];
            }
            __syncwarp();
            const int r = r0 + lane;
#pragma unroll 4
            for (int i = 0; i < 32; ++i) {
              const int q = q0 + i;
              if (q < R && r < C) {
                CT x[A];
#pragma unroll
                for (int k = 0; k < A; ++k)
                  x[k] = to_ct<DT>(tr[k] ? tile[(k * 32 + lane) * 33 + i] : __ldcg(in[k] + (q * s0[1 + k] + r * s1[1 + k])));
                out[q * s0[0] + r] = from_ct<DT>(fast_eval<DT>(f, x));
              }
            }
            __syncwarp();
          }
          return;
        }
        constexpr int U2F = 16;
        const int64_t stepf = (int64_t)c->nthreads * U2F;
        for (int64_t e0 = lo + c->tid; e0 < hi; e0 += stepf) {
          CT x[U2F][A];
          int32_t oo[U2F];
#pragma unroll
          for (int u = 0; u < U2F; ++u) {
            const int64_t e = e0 + (int64_t)u * c->nthreads;
            if (e < hi) {
              const uint32_t q = fd.div((uint32_t)e), r = (uint32_t)e - q * fd.d;
              oo[u] = (int32_t)q * s0[0] + (int32_t)r * s1[0];
#pragma unroll
              for (int k = 0; k < A; ++k) x[u][k] = to_ct<DT>(__ldcg(in[k] + ((int32_t)q * s0[1 + k] + (int32_t)r * s1[1 + k])));
            }
          }
#pragma unroll
          for (int u = 0; u < U2F; ++u) {
            const int64_t e = e0 + (int64_t)u * c->nthreads;
            if (e < hi) out[oo[u]] = from_ct<DT>(fast_eval<DT>(f, x[u]));
          }
        }
        return;
      }
    }
    constexpr int U2 = 8;
    const int64_t step = (int64_t)c->nthreads * U2;
    for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
      double x[U2][A];
      int64_t oo[U2];
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) {
          const uint32_t q = fd.div((uint32_t)e), r = (uint32_t)e - q * fd.d;
          oo[u] = (int64_t)q * st0[0] + (int64_t)r * st1[0];
#pragma unroll
          for (int k = 0; k < A; ++k) x[u][k] = DT_<DT>::gload(in[k] + (int64_t)q * st0[1 + k] + (int64_t)r * st1[1 + k]);
        }
      }
#pragma unroll
      for (int u = 0; u < U2; ++u) {
        const int64_t e = e0 + (int64_t)u * c->nthreads;
        if (e < hi) DT_<DT>::store(out + oo[u], f(x[u]));
      }
    }
    return;
  }
  // U elements per thread per round, all loads issued before any use, so a
  // round costs one memory latency instead of U
  constexpr int U = 4;
  const int64_t step = (int64_t)c->nthreads * U;
  for (int64_t e0 = lo + c->tid; e0 < hi; e0 += step) {
    int64_t off[U][1 + A];
    double x[U][A];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * c->nthreads;
      if (e < hi) {
        space_offsets(s, (uint32_t)e, off[u]);
#pragma unroll
        for (int k = 0; k < A; ++k) x[u][k] = DT_<DT>::gload(in[k] + off[u][1 + k]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * c->nthreads;
      if (e < hi) DT_<DT>::store(out + off[u][0], f(x[u]));
    }
  }
}

// Checks in the reference order (ops.hpp:133-153), then dispatch on dtype.
template <int DT, class F>
__device__ __forceinline__ void ew_dense_any(const gpuos_task* t, const Ctx* c, int64_t n, F f) {
  ew_dense<DT>(t, c, n, f);
}
template <class F>
__device__ __forceinline__ bool ew_dense_dispatch(const gpuos_task* t, const Ctx* c, int dt, int64_t n, F f) {
  switch (dt) {
    case GPUOS_F32: ew_dense_any<GPUOS_F32>(t, c, n, f); return true;
    case GPUOS_F64: ew_dense_any<GPUOS_F64>(t, c, n, f); return true;
    case GPUOS_I32: ew_dense_any<GPUOS_I32>(t, c, n, f); return true;
    case GPUOS_F16: ew_dense_any<GPUOS_F16>(t, c, n, f); return true;
    case GPUOS_BF16: ew_dense_any<GPUOS_BF16>(t, c, n, f); return true;
    default: return false;
  }
}

template <class F>
__device__ int ew_body(const gpuos_task* t, const Ctx* c, bool allow_int) {
  constexpr int A = F::A;
  if (t->n_inputs != A) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  if (c->flags & kPlanDenseSame) {
    // planned: same dtype/shape, dense, bound; only the dtype class and the
    // size ceiling remain to check (ops.hpp:133-153 order preserved)
    const int dt = out.dtype;
    if (!allow_int && dt == GPUOS_I32) return GPUOS_DTYPE_MISMATCH;
    const int64_t n = numel(out);
    if (n == 0) return GPUOS_OK;
    if (n < ((int64_t)1 << 31)) {
      F f;
      return ew_dense_dispatch(t, c, dt, n, f) ? GPUOS_OK : GPUOS_DTYPE_MISMATCH;
    }
  }
  if (!allow_int && out.dtype == GPUOS_I32) return GPUOS_DTYPE_MISMATCH;
  for (int k = 0; k < A; ++k)
    if (t->views[1 + k].dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  const int64_t n = numel(out);
  if (n == 0) return GPUOS_OK;
  if (n >= (int64_t)1 << 31) return GPUOS_TOO_LARGE;
  int64_t st[A][GPUOS_MAX_RANK];
  for (int k = 0; k < A; ++k) {
    if (!broadcast_strides(t->views[1 + k], out, st[k])) return GPUOS_INCOMPATIBLE_SHAPES;
    const int b = bind_code(t->views[1 + k]);
    if (b) return b;
  }
  const int b = bind_code(out);
  if (b) return b;
  F f;
  // common case first: every operand dense with the output's shape, so the
  // strided iteration space (and its divmod setup) is not needed
  bool simple = dense_view(out);
  for (int k = 0; k < A && simple; ++k) simple = same_shape(t->views[1 + k], out) && dense_view(t->views[1 + k]);
  if (simple) return ew_dense_dispatch(t, c, out.dtype, n, f) ? GPUOS_OK : GPUOS_DTYPE_MISMATCH;
  if (dense_view(out)) {
    // every input flattens to one stride against the dense output (rank-0
    // scalars, stride-k views, ...): the rank-1 loop, no iteration space
    int64_t fs[1 + A];
    fs[0] = 1;
    bool flat = true;
#pragma unroll
    for (int k = 0; k < A; ++k) flat = flat && flat_stride(t->views[1 + k], out, &fs[1 + k]);
    if (flat) {
      switch (out.dtype) {
        case GPUOS_F32: ew_rank1<GPUOS_F32>(t, c, n, f, fs); return GPUOS_OK;
        case GPUOS_F64: ew_rank1<GPUOS_F64>(t, c, n, f, fs); return GPUOS_OK;
        case GPUOS_I32: ew_rank1<GPUOS_I32>(t, c, n, f, fs); return GPUOS_OK;
        case GPUOS_F16: ew_rank1<GPUOS_F16>(t, c, n, f, fs); return GPUOS_OK;
        case GPUOS_BF16: ew_rank1<GPUOS_BF16>(t, c, n, f, fs); return GPUOS_OK;
        default: return GPUOS_DTYPE_MISMATCH;
      }
    }
  }
  Space s;
  build_space(s, out, A, st);
  switch (out.dtype) {
#define GPUOS_EW_CASE(DT)                        \
  case DT:                                       \
    if (s.dense)                                 \
      ew_dense_any<DT>(t, c, n, f);              \
    else                                         \
      ew_strided<DT>(t, c, s, n, f);             \
    break;
    GPUOS_EW_CASE(GPUOS_F32)
    GPUOS_EW_CASE(GPUOS_F64)
    GPUOS_EW_CASE(GPUOS_I32)
    GPUOS_EW_CASE(GPUOS_F16)
    GPUOS_EW_CASE(GPUOS_BF16)
#undef GPUOS_EW_CASE
    default: return GPUOS_DTYPE_MISMATCH;
  }
  return GPUOS_OK;
}

// General path: every reference check, every dtype, strided/broadcast.
template <class F>
__device__ __noinline__ int ew_general(const gpuos_task* t, const Ctx* c, bool allow_int) {
  return ew_body<F>(t, c, allow_int);
}

// Entry points in the jump table.  A planned dense f32 task (the common small
// op) runs its loop right here; everything else goes through ew_general.
// Keeping the heavy general path out of line keeps these functions' register
// footprint -- and so the callee-saved spills of every indirect call -- small
// (measured: tools/probe/body_bench.cu).
template <class F>
__device__ __forceinline__ int ew_entry(const gpuos_task* t, const Ctx* c, bool allow_int) {
  if ((c->flags & kPlanDenseSame) && t->n_inputs == F::A && t->views[0].dtype == GPUOS_F32) {
    const int64_t n = numel(t->views[0]);
    if (n > 0 && n < ((int64_t)1 << 31)) {
      F f;
      // (cp.async.bulk + mbarrier streaming variants were measured twice and
      // dropped: slower at 4K-64K elements in round 1; a two-stage pipelined
      // one hung on the box in round 2, while this register path already
      // streams 64K-element tasks at 5.0 TB/s, profiles/r02_*)
      ew_dense<GPUOS_F32>(t, c, n, f);
      return GPUOS_OK;
    }
  }
  return ew_general<F>(t, c, allow_int);
}

#ifndef GPUOS_JIT_TU  // a natively compiled injected op links against these; it must not redefine them
__device__ __noinline__ int op_add(const gpuos_task* t, const Ctx* c) { return ew_entry<FAdd>(t, c, true); }
__device__ __noinline__ int op_mul(const gpuos_task* t, const Ctx* c) { return ew_entry<FMul>(t, c, true); }
__device__ __noinline__ int op_relu(const gpuos_task* t, const Ctx* c) { return ew_entry<FRelu>(t, c, true); }
__device__ __noinline__ int op_gelu(const gpuos_task* t, const Ctx* c) { return ew_general<FGelu>(t, c, false); }
#endif

// ---------------------------------------------------------------------------
// Injected operators: a verified stack-machine program evaluated in double per
// element over broadcast inputs.  Program layout in HBM: ProgramHeader then
// n_instr gpuos_instr.  (Live injection path: no module load.)
// ---------------------------------------------------------------------------

__device__ __forceinline__ double run_program(const gpuos_instr* code, int n_instr, const double* in) {
  double stack[GPUOS_MAX_STACK];
  int sp = 0;
  for (int pc = 0; pc < n_instr; ++pc) {
    const gpuos_instr ins = code[pc];
    switch (ins.op) {
      case GPUOS_BC_PUSH_CONST: stack[sp++] = ins.value; break;
      case GPUOS_BC_LOAD_IN: stack[sp++] = in[ins.k]; break;
      case GPUOS_BC_ADD: --sp; stack[sp - 1] = __dadd_rn(stack[sp - 1], stack[sp]); break;
      case GPUOS_BC_SUB: --sp; stack[sp - 1] = __dsub_rn(stack[sp - 1], stack[sp]); break;
      case GPUOS_BC_MUL: --sp; stack[sp - 1] = __dmul_rn(stack[sp - 1], stack[sp]); break;
      case GPUOS_BC_DIV: --sp; stack[sp - 1] = __ddiv_rn(stack[sp - 1], stack[sp]); break;
      case GPUOS_BC_NEG: stack[sp - 1] = -stack[sp - 1]; break;
      case GPUOS_BC_EXP: stack[sp - 1] = exp(stack[sp - 1]); break;
      case GPUOS_BC_TANH: stack[sp - 1] = tanh(stack[sp - 1]); break;
      case GPUOS_BC_MAX: {  // binop_max: a < b ? b : a (expr.hpp:134)
        --sp;
        const double a = stack[sp - 1], b = stack[sp];
        stack[sp - 1] = a < b ? b : a;
        break;
      }
      case GPUOS_BC_MIN: {  // binop_min: b < a ? b : a (expr.hpp:135)
        --sp;
        const double a = stack[sp - 1], b = stack[sp];
        stack[sp - 1] = b < a ? b : a;
        break;
      }
      case GPUOS_BC_ABS: stack[sp - 1] = fabs(stack[sp - 1]); break;
      case GPUOS_BC_SQRT: stack[sp - 1] = __dsqrt_rn(stack[sp - 1]); break;
      case GPUOS_BC_NARROW: stack[sp - 1] = narrow_any(ins.k, stack[sp - 1]); break;
      default: return stack[sp - 1];  // STORE_OUT
    }
  }
  return stack[sp > 0 ? sp - 1 : 0];
}

template <int DT>
__device__ void program_loop(const gpuos_task* t, const Ctx* c, const Space& s, int64_t n,
                             const gpuos_instr* code, int n_instr, int arity) {
  typedef typename DT_<DT>::T T;
  T* out = (T*)t->views[0].addr;
  const T* in[GPUOS_MAX_INPUTS];
  for (int k = 0; k < arity; ++k) in[k] = (const T*)t->views[1 + k].addr;
  int64_t lo, hi;
  part_range(n, c->part, c->nparts, 1, &lo, &hi);
  for (int64_t e = lo + c->tid; e < hi; e += c->nthreads) {
    int64_t off[1 + GPUOS_MAX_INPUTS];
    if (s.dense) {
      for (int k = 0; k <= arity; ++k) off[k] = e;
    } else {
      space_offsets(s, (uint32_t)e, off);
    }
    double x[GPUOS_MAX_INPUTS];
    for (int k = 0; k < arity; ++k) x[k] = DT_<DT>::gload(in[k] + off[1 + k]);
    DT_<DT>::store(out + off[0], run_program(code, n_instr, x));
  }
}

#ifndef GPUOS_JIT_TU
// Checks in load_module's order (opcompiler.hpp:72-101).
__device__ __noinline__ int op_program(const gpuos_task* t, const Ctx* c) {
  const ProgramHeader* hp = (const ProgramHeader*)c->aux;
  if (hp == nullptr) return GPUOS_VERIFY_ERROR;
  ProgramHeader hh;  // L2 reads (see the coherence rule in dev_common.cuh)
  hh.n_instr = __ldcg(&hp->n_instr);
  hh.arity = __ldcg(&hp->arity);
  hh.dtype = __ldcg(&hp->dtype);
  const ProgramHeader* h = &hh;
  const int arity = h->arity;
  if (t->n_inputs != arity) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  if (out.dtype != h->dtype) return GPUOS_DTYPE_MISMATCH;
  const int64_t n = numel(out);
  if (n == 0) return GPUOS_OK;
  if (n >= (int64_t)1 << 31) return GPUOS_TOO_LARGE;
  Space s;
  if (c->flags & kPlanDenseSame) {
    s.dense = true;  // planned: dtypes, shapes, binds already known good
    s.nops = arity + 1;
    s.rank = 0;
  } else {
    int64_t st[GPUOS_MAX_INPUTS][GPUOS_MAX_RANK];
    for (int k = 0; k < arity; ++k) {
      if (t->views[1 + k].dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
      if (!broadcast_strides(t->views[1 + k], out, st[k])) return GPUOS_INCOMPATIBLE_SHAPES;
      const int b = bind_code(t->views[1 + k]);
      if (b) return b;
    }
    const int b = bind_code(out);
    if (b) return b;
    build_space(s, out, arity, st);
  }
  // stage the program in shared memory (<= GPUOS_MAX_PROGRAM instructions)
  const int n_instr = (int)h->n_instr;
  gpuos_instr* code = (gpuos_instr*)c->smem;
  const uint4* src = (const uint4*)(hp + 1);
  for (int i = c->tid; i < n_instr; i += c->nthreads) reinterpret_cast<uint4*>(code)[i] = __ldcg(src + i);
  group_sync(c);
  switch (out.dtype) {
    case GPUOS_F32: program_loop<GPUOS_F32>(t, c, s, n, code, n_instr, arity); break;
    case GPUOS_F64: program_loop<GPUOS_F64>(t, c, s, n, code, n_instr, arity); break;
    case GPUOS_I32: program_loop<GPUOS_I32>(t, c, s, n, code, n_instr, arity); break;
    case GPUOS_F16: program_loop<GPUOS_F16>(t, c, s, n, code, n_instr, arity); break;
    case GPUOS_BF16: program_loop<GPUOS_BF16>(t, c, s, n, code, n_instr, arity); break;
    default: break;
  }
  group_sync(c);  // program scratch is reused by the next task
  return GPUOS_OK;
}

// ---------------------------------------------------------------------------
// kv_append: inputs {new_k, new_v, v_cache}, output k_cache, scalars[0] = cursor
// (ops.hpp:544-589).  A bit-exact copy through the double load/store path.
// ---------------------------------------------------------------------------
__device__ __noinline__ int op_kv_append(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 3) return GPUOS_ARITY_ERROR;
  if (t->n_scalars == 0) return GPUOS_ARITY_ERROR;
  const gpuos_view& kc = t->views[0];
  const gpuos_view& nk = t->views[1];
  const gpuos_view& nv = t->views[2];
  const gpuos_view& vc = t->views[3];
  if (kc.rank != 3 || vc.rank != 3 || nk.rank != 2 || nv.rank != 2) return GPUOS_SHAPE_MISMATCH;
  const int h = kc.extents[0], cap = kc.extents[1], d = kc.extents[2];
  if (!same_shape(vc, kc)) return GPUOS_SHAPE_MISMATCH;
  if (nk.extents[0] != h || nk.extents[1] != d || nv.extents[0] != h || nv.extents[1] != d)
    return GPUOS_SHAPE_MISMATCH;
  if (nk.dtype != kc.dtype || nv.dtype != vc.dtype || vc.dtype != kc.dtype) return GPUOS_DTYPE_MISMATCH;
  const double cs = t->scalars[0];
  // static_cast<int64_t>(double): truncation; NaN/out-of-range land outside [0, cap)
  const int64_t cursor = (cs > -9.2e18 && cs < 9.2e18) ? (int64_t)cs : (int64_t)-1;
  if (cursor < 0 || cursor >= cap) return GPUOS_CACHE_FULL;
  int b;
  if ((b = bind_code(kc)) || (b = bind_code(vc)) || (b = bind_code(nk)) || (b = bind_code(nv))) return b;
  const int dt = kc.dtype;
  const int64_t total = (int64_t)h * d;
  int64_t lo, hi;
  part_range(total, c->part, c->nparts, 1, &lo, &hi);
  for (int64_t e = lo + c->tid; e < hi; e += c->nthreads) {
    const int64_t head = e / d, j = e % d;
    const int64_t ko = head * kc.strides[0] + cursor * kc.strides[1] + j * kc.strides[2];
    const int64_t vo = head * vc.strides[0] + cursor * vc.strides[1] + j * vc.strides[2];
    const int64_t no = head * nk.strides[0] + j * nk.strides[1];
    const int64_t mo = head * nv.strides[0] + j * nv.strides[1];
    store_any(dt, (char*)kc.addr, ko, load_any(dt, (const char*)nk.addr, no));
    store_any(dt, (char*)vc.addr, vo, load_any(dt, (const char*)nv.addr, mo));
  }
  return GPUOS_OK;
}

#endif  // GPUOS_JIT_TU

// ---------------------------------------------------------------------------
// Natively compiled injected operators: the host generates a functor F from
// the verified program (straight-line code, same fp64 operations in the same
// order, one rounding on store) and instantiates jit_body<F, DT> in an NVRTC
// translation unit.  Checks in op_program's order (opcompiler.hpp:72-101), so
// a promoted op returns exactly what its device program returns.
// ---------------------------------------------------------------------------
template <class F, int DT>
__device__ __forceinline__ int jit_body(const gpuos_task* t, const Ctx* c) {
  constexpr int A = F::A;
  if (t->n_inputs != A) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  if (out.dtype != DT) return GPUOS_DTYPE_MISMATCH;
  const int64_t n = numel(out);
  if (n == 0) return GPUOS_OK;
  if (n >= (int64_t)1 << 31) return GPUOS_TOO_LARGE;
  F f;
  if (c->flags & kPlanDenseSame) {
    ew_dense<DT>(t, c, n, f);
    return GPUOS_OK;
  }
  int64_t st[A > 0 ? A : 1][GPUOS_MAX_RANK];
  for (int k = 0; k < A; ++k) {
    if (t->views[1 + k].dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
    if (!broadcast_strides(t->views[1 + k], out, st[k])) return GPUOS_INCOMPATIBLE_SHAPES;
    const int b = bind_code(t->views[1 + k]);
    if (b) return b;
  }
  const int b = bind_code(out);
  if (b) return b;
  Space s;
  build_space(s, out, A, st);
  if (s.dense) ew_dense<DT>(t, c, n, f);
  else ew_strided<DT>(t, c, s, n, f);
  return GPUOS_OK;
}

}  // namespace gdev
