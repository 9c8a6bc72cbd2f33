// Matrix and attention task bodies on CUDA cores in fp64: matmul_small /
// vecmat (reference ops.hpp:363-433), single-query sdpa (ops.hpp:441-498) and
// rope (ops.hpp:503-537).
//
// Accumulation order matches the reference exactly (ascending k, one rounding
// per product and per add).  For f32/f16/bf16 operands every product is exact
// in fp64, so a DFMA equals the reference's separate multiply and add and is
// used; f64/i32 operands use __dmul_rn + __dadd_rn.  bf16/f16 matmuls run on
// the tensor cores (tcgen05, ops_umma.cuh) when the executing group has TMEM.
#pragma once

#include "dev_common.cuh"
#include "ops_umma.cuh"

namespace gdev {

__device__ __forceinline__ bool exact_products(int dt) {
  return dt == GPUOS_F32 || dt == GPUOS_F16 || dt == GPUOS_BF16;
}
__device__ __forceinline__ double mac(double acc, double a, double b, bool exact) {
  return exact ? fma(a, b, acc) : __dadd_rn(acc, __dmul_rn(a, b));
}

// ---- matmul: a (m,k) x b (k,n) -> out (m,n) ----
constexpr int kTM = 64, kTN = 64, kTK = 32;

// Staging of one k-step for the 4x4-per-thread grid (TM = nthreads/4 rows):
// every thread issues its loads back to back into registers (raw element
// type, 8 per batch), then converts and writes shared memory, so a k-step
// costs one memory latency per batch instead of one per element.  Same
// values, same order of accumulation: results are unchanged.
// One k-step of the 4x4 register tile.  The fma/mul-add choice is a template
// parameter so the loop carries one form, and the tiles are read through
// shared-window addresses: with a runtime select and 64-bit generic
// pointers, ptxas spilled half of the 16 accumulators inside this loop.
template <bool kExact>
__device__ __forceinline__ void mm_kloop(double (&acc)[4][4], const double* As, const double* Bs, int ty, int tx, int R,
                                         int kmax) {
  const uint32_t as = (uint32_t)__cvta_generic_to_shared(As) + (uint32_t)(ty * (kTK + 1)) * 8u;
  const uint32_t bs = (uint32_t)__cvta_generic_to_shared(Bs) + (uint32_t)tx * 8u;
  const uint32_t astep = (uint32_t)(R * (kTK + 1)) * 8u;
  for (int kk = 0; kk < kmax; ++kk) {
    double av[4], bv[4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(av[r]) : "r"(as + r * astep + (uint32_t)kk * 8u));
#pragma unroll
    for (int q = 0; q < 4; ++q)
      asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bv[q]) : "r"(bs + (uint32_t)(kk * (kTN + 1) + 16 * q) * 8u));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = mac(acc[r][q], av[r], bv[q], kExact);
  }
}

struct MatStage {
  const char* ap;
  const char* bp;
  int64_t sa0, sa1, sb0, sb1;
  int m, n, k, i0, j0, k0;
  double* As;
  double* Bs;
};
template <int DT>
__device__ __forceinline__ void stage_grid(const MatStage& s, const Ctx* c) {
  typedef typename DT_<DT>::T T;
  constexpr int kBatch = 8;
  const T* A = reinterpret_cast<const T*>(s.ap);
  const T* B = reinterpret_cast<const T*>(s.bp);
  const int nt = c->nthreads, tid = c->tid;
  // A: TM x kTK = 8 * nt elements, exactly one batch per thread
  {
    T v[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const int e = tid + nt * q;
      const int gi = s.i0 + e / kTK, gk = s.k0 + e % kTK;
      v[q] = (gi < s.m && gk < s.k) ? __ldcg(A + gi * s.sa0 + gk * s.sa1) : T(0);
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const int e = tid + nt * q;
      s.As[(e / kTK) * (kTK + 1) + e % kTK] = DT_<DT>::load(&v[q]);
    }
  }
  // B: kTK x kTN = 2048 elements, 2048 / nt / 8 batches per thread
  for (int b0 = 0; b0 < kTK * kTN; b0 += nt * kBatch) {
    T v[kBatch];
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const int e = b0 + tid + nt * q;
      const int gk = s.k0 + e / kTN, gj = s.j0 + e % kTN;
      v[q] = (e < kTK * kTN && gk < s.k && gj < s.n) ? __ldcg(B + gk * s.sb0 + gj * s.sb1) : T(0);
    }
#pragma unroll
    for (int q = 0; q < kBatch; ++q) {
      const int e = b0 + tid + nt * q;
      if (e < kTK * kTN) s.Bs[(e / kTN) * (kTN + 1) + e % kTN] = DT_<DT>::load(&v[q]);
    }
  }
}

__device__ __noinline__ int op_matmul(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 2) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& a = t->views[1];
  const gpuos_view& b = t->views[2];
  if (a.dtype != out.dtype || b.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (a.rank != 2 || b.rank != 2 || out.rank != 2) return GPUOS_SHAPE_MISMATCH;
  const int m = a.extents[0], k = a.extents[1], n = b.extents[1];
  if (b.extents[0] != k) return GPUOS_SHAPE_MISMATCH;
  if (out.extents[0] != m || out.extents[1] != n) return GPUOS_SHAPE_MISMATCH;
  if (!(c->flags & GPUOS_FLAG_UNCAPPED) &&
      (m > GPUOS_SMALL_MATMUL_MAX_DIM || k > GPUOS_SMALL_MATMUL_MAX_DIM || n > GPUOS_SMALL_MATMUL_MAX_DIM))
    return GPUOS_TOO_LARGE;
  int bc;
  if ((bc = bind_code(a)) || (bc = bind_code(b)) || (bc = bind_code(out))) return bc;
  const int dt = out.dtype;
  // 16-bit floats: tensor cores (tcgen05, ops_umma.cuh) when the group holds TMEM
  if ((dt == GPUOS_BF16 || dt == GPUOS_F16) && c->tmem != kNoTmem && c->smem_bytes >= 2 * (int)kUmmaTileBytes &&
      m > 0 && n > 0 && k > 0)
    return matmul_umma(a, b, out, m, k, n, c);
  const bool exact = exact_products(dt);
  const char* ap = (const char*)a.addr;
  const char* bp = (const char*)b.addr;
  char* op = (char*)out.addr;
  const int64_t sa0 = a.strides[0], sa1 = a.strides[1], sb0 = b.strides[0], sb1 = b.strides[1];
  const int64_t so0 = out.strides[0], so1 = out.strides[1];
  double* As = (double*)c->smem;             // [kTM][kTK+1]
  double* Bs = As + kTM * (kTK + 1);         // [kTK][kTN+1]
  const int nt = c->nthreads;
  // Thread grid: (nt/16) x 16 threads, 4x4 outputs each (rows ty + R*r, cols
  // tx + 16q), so a tile is (4*nt/16) x 64: 64x64 for a 256-thread group,
  // 32x64 for the worker's 128-thread groups.  Other group sizes use the
  // element loop with a tile small enough that 16 outputs per thread cover it.
  const bool grid = (nt % 16 == 0) && nt >= 16 && nt <= 256;
  const int R = nt / 16;
  const int TM = grid ? 4 * R : ((nt * 16) / kTN < kTM ? ((nt * 16) / kTN > 0 ? (nt * 16) / kTN : 1) : kTM);
  const int ntm = (m + TM - 1) / TM, ntn = (n + kTN - 1) / kTN;
  int64_t tlo, thi;
  part_range((int64_t)ntm * ntn, c->part, c->nparts, 1, &tlo, &thi);
  const int ty = c->tid >> 4, tx = c->tid & 15;
  for (int64_t tile = tlo; tile < thi; ++tile) {
    const int i0 = (int)(tile / ntn) * TM, j0 = (int)(tile % ntn) * kTN;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[r][q] = 0.0;
    for (int k0 = 0; k0 < k; k0 += kTK) {
      bool staged = false;
      if (grid) {
        const MatStage st{ap, bp, sa0, sa1, sb0, sb1, m, n, k, i0, j0, k0, As, Bs};
        switch (dt) {
          case GPUOS_F32: stage_grid<GPUOS_F32>(st, c); staged = true; break;
          case GPUOS_F64: stage_grid<GPUOS_F64>(st, c); staged = true; break;
          case GPUOS_I32: stage_grid<GPUOS_I32>(st, c); staged = true; break;
          default: break;
        }
      }
      if (!staged) {
        for (int e = c->tid; e < TM * kTK; e += nt) {
          const int i = e / kTK, kk = e % kTK;
          const int gi = i0 + i, gk = k0 + kk;
          As[i * (kTK + 1) + kk] = (gi < m && gk < k) ? load_any(dt, ap, gi * sa0 + gk * sa1) : 0.0;
        }
        for (int e = c->tid; e < kTK * kTN; e += nt) {
          const int kk = e / kTN, j = e % kTN;
          const int gk = k0 + kk, gj = j0 + j;
          Bs[kk * (kTN + 1) + j] = (gk < k && gj < n) ? load_any(dt, bp, gk * sb0 + gj * sb1) : 0.0;
        }
      }
      group_sync(c);
      const int kmax = (k - k0) < kTK ? (k - k0) : kTK;
      if (grid) {
        if (exact) mm_kloop<true>(acc, As, Bs, ty, tx, R, kmax);
        else mm_kloop<false>(acc, As, Bs, ty, tx, R, kmax);
      } else {
        // each thread owns tile elements e = tid + nt*s (s < 16)
        for (int s = 0; s < 16; ++s) {
          const int e = c->tid + nt * s;
          if (e >= TM * kTN) break;
          const int i = e / kTN, j = e % kTN;
          double v = acc[s >> 2][s & 3];
          for (int kk = 0; kk < kmax; ++kk) v = mac(v, As[i * (kTK + 1) + kk], Bs[kk * (kTN + 1) + j], exact);
          acc[s >> 2][s & 3] = v;
        }
      }
      group_sync(c);
    }
    if (grid) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int gi = i0 + ty + R * r, gj = j0 + tx + 16 * q;
          if (gi < m && gj < n) store_any(dt, op, gi * so0 + gj * so1, acc[r][q]);
        }
    } else {
      for (int s = 0; s < 16; ++s) {
        const int e = c->tid + nt * s;
        if (e >= TM * kTN) break;
        const int gi = i0 + e / kTN, gj = j0 + e % kTN;
        if (gi < m && gj < n) store_any(dt, op, gi * so0 + gj * so1, acc[s >> 2][s & 3]);
      }
    }
  }
  return GPUOS_OK;
}

// ---- vecmat: v (k) x mat (k,n) -> out (n) ----
__device__ __noinline__ int op_vecmat(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 2) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& v = t->views[1];
  const gpuos_view& mt = t->views[2];
  if (v.dtype != out.dtype || mt.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (v.rank != 1 || mt.rank != 2 || out.rank != 1) return GPUOS_SHAPE_MISMATCH;
  const int k = v.extents[0], n = mt.extents[1];
  if (mt.extents[0] != k || out.extents[0] != n) return GPUOS_SHAPE_MISMATCH;
  if (!(c->flags & GPUOS_FLAG_UNCAPPED) && (k > GPUOS_SMALL_MATMUL_MAX_DIM || n > GPUOS_SMALL_MATMUL_MAX_DIM))
    return GPUOS_TOO_LARGE;
  int bc;
  if ((bc = bind_code(v)) || (bc = bind_code(mt)) || (bc = bind_code(out))) return bc;
  const int dt = out.dtype;
  const bool exact = exact_products(dt);
  int64_t lo, hi;
  part_range(n, c->part, c->nparts, 1, &lo, &hi);
  for (int64_t j = lo + c->tid; j < hi; j += c->nthreads) {
    double acc = 0.0;
    for (int p = 0; p < k; ++p)
      acc = mac(acc, load_any(dt, (const char*)v.addr, (int64_t)p * v.strides[0]),
                load_any(dt, (const char*)mt.addr, (int64_t)p * mt.strides[0] + j * mt.strides[1]), exact);
    store_any(dt, (char*)out.addr, j * out.strides[0], acc);
  }
  return GPUOS_OK;
}

// ---- sdpa: q (h,d), k (h,t,d), v (h,t,d) -> out (h,d) ----
__device__ __forceinline__ double nan_skip_max(double a, double b) {
  if (b != b) return a;
  if (a != a) return b;
  return a < b ? b : a;
}

// Batched-head sdpa: the q rows and the scores of up to kSdpaHB heads sit in
// shared memory; each weight e_i / denom is formed once per key instead of
// once per (key, column); the output columns of every head in the batch
// accumulate together, two ascending-key chains per thread with eight keys
// of v in flight.  Operands are held in their storage type until use (a
// double per element in flight spilled the unrolled loops to local memory).
// Every value is computed in the reference's order (ascending j per score,
// ascending i per output column, ops.hpp:441-498).
constexpr int kSdpaHB = 8;
#ifndef GPUOS_SDPA_VU
#define GPUOS_SDPA_VU 4
#endif
constexpr int kSdpaVU = GPUOS_SDPA_VU;  // keys of v in flight per round (pass 3)
#ifndef GPUOS_SDPA_KU
#define GPUOS_SDPA_KU 8
#endif
constexpr int kSdpaKU = GPUOS_SDPA_KU;  // key elements in flight per round (pass 1)
__device__ __forceinline__ int sdpa_heads_per_batch(const Ctx* c, int d, int tl) {
  const int nw = c->nthreads >> 5;
  if (d > 256 || nw > 8 || d <= 0) return 0;
  const int fixed = 8 * kSdpaHB + 2 * kSdpaHB + kSdpaHB * d;  // doubles: red, stats, q rows
  const int avail = c->smem_bytes / 8 - fixed;
  int hb = kSdpaHB;
  if (avail / tl < hb) hb = avail / tl;
  if ((2 * c->nthreads) / d < hb) hb = (2 * c->nthreads) / d;
  return hb;
}
template <int DT>
__device__ __noinline__ void sdpa_batched(const gpuos_task* t, const Ctx* c, int hb, int64_t hlo, int64_t hhi,
                                          double scale) {
  typedef typename DT_<DT>::T T;
  const gpuos_view& out = t->views[0];
  const gpuos_view& q = t->views[1];
  const gpuos_view& kk = t->views[2];
  const gpuos_view& vv = t->views[3];
  const int d = q.extents[1], tl = kk.extents[1];
  const bool exact = exact_products(DT);
  const int nw = c->nthreads >> 5;
  double* red = (double*)c->smem;
  double* stat = red + 8 * kSdpaHB;  // [0, kSdpaHB): max, [kSdpaHB, 2 kSdpaHB): denominator
  double* qs = stat + 2 * kSdpaHB;
  double* sc = qs + kSdpaHB * d;
  const T* qp = (const T*)q.addr;
  const T* kp = (const T*)kk.addr;
  const T* vp = (const T*)vv.addr;
  const int64_t ks0 = kk.strides[0], ks1 = kk.strides[1], ks2 = kk.strides[2];
  for (int64_t h0 = hlo; h0 < hhi; h0 += hb) {
    const int nb = (int)((hhi - h0) < hb ? (hhi - h0) : hb);
    for (int e = c->tid; e < nb * d; e += c->nthreads) {
      const int hh = e / d, j = e - hh * d;
      qs[e] = DT_<DT>::gload(qp + (h0 + hh) * q.strides[0] + (int64_t)j * q.strides[1]);
    }
    group_sync(c);
    // pass 1: scores and per-head max; kSdpaKU key elements in flight per round
#pragma unroll 1
    for (int hh = 0; hh < nb; ++hh) {
      const T* kb = kp + (h0 + hh) * ks0;
      const double* qr = qs + hh * d;
      double mx = -INFINITY;
      for (int i = c->tid; i < tl; i += c->nthreads) {
        const T* kr = kb + (int64_t)i * ks1;
        double dot = 0.0;
        for (int j0 = 0; j0 < d; j0 += kSdpaKU) {
          T kv[kSdpaKU];
#pragma unroll
          for (int u = 0; u < kSdpaKU; ++u)
            if (j0 + u < d) kv[u] = __ldcg(kr + (int64_t)(j0 + u) * ks2);
#pragma unroll
          for (int u = 0; u < kSdpaKU; ++u)
            if (j0 + u < d) dot = mac(dot, qr[j0 + u], DT_<DT>::load(&kv[u]), exact);
        }
        const double sv = __dmul_rn(scale, dot);
        sc[hh * tl + i] = sv;
        mx = nan_skip_max(mx, sv);
      }
      for (int o = 16; o > 0; o >>= 1) mx = nan_skip_max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((c->tid & 31) == 0) red[(c->tid >> 5) * kSdpaHB + hh] = mx;
    }
    group_sync(c);
    if (c->tid < nb) {
      double mx = -INFINITY;
      for (int w = 0; w < nw; ++w) mx = nan_skip_max(mx, red[w * kSdpaHB + c->tid]);
      stat[c->tid] = mx;
    }
    group_sync(c);
    // pass 2: e_i = exp(s_i - max) and the per-head denominators
#pragma unroll 1
    for (int hh = 0; hh < nb; ++hh) {
      const double mx = stat[hh];
      double sum = 0.0;
      for (int i = c->tid; i < tl; i += c->nthreads) {
        const double ev = exp(__dsub_rn(sc[hh * tl + i], mx));
        sc[hh * tl + i] = ev;
        sum += ev;
      }
      sum = warp_sum(sum);
      if ((c->tid & 31) == 0) red[(c->tid >> 5) * kSdpaHB + hh] = sum;
    }
    group_sync(c);
    if (c->tid < nb) {
      double sum = 0.0;
      for (int w = 0; w < nw; ++w) sum += red[w * kSdpaHB + c->tid];
      stat[kSdpaHB + c->tid] = sum;
    }
    group_sync(c);
    // weights w_i = e_i / denom, once per key
    for (int e = c->tid; e < nb * tl; e += c->nthreads) sc[e] = __ddiv_rn(sc[e], stat[kSdpaHB + e / tl]);
    group_sync(c);
    // pass 3: out[hh][j] = sum_i w_i * v[i][j], ascending i
    int ph[2], pj[2];
    double acc[2] = {0.0, 0.0};
    const T* vb[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int pidx = c->tid + r * c->nthreads;
      ph[r] = pidx < nb * d ? pidx / d : -1;
      pj[r] = pidx < nb * d ? pidx - ph[r] * d : 0;
      vb[r] = vp + (ph[r] >= 0 ? (h0 + ph[r]) * vv.strides[0] + (int64_t)pj[r] * vv.strides[2] : 0);
    }
    const int64_t vstep = vv.strides[1];
    for (int i0 = 0; i0 < tl; i0 += kSdpaVU) {
      T vr[kSdpaVU][2];
#pragma unroll
      for (int u = 0; u < kSdpaVU; ++u)
#pragma unroll
        for (int r = 0; r < 2; ++r)
          if (ph[r] >= 0 && i0 + u < tl) vr[u][r] = __ldcg(vb[r] + (int64_t)(i0 + u) * vstep);
#pragma unroll
      for (int u = 0; u < kSdpaVU; ++u)
#pragma unroll
        for (int r = 0; r < 2; ++r)
          if (ph[r] >= 0 && i0 + u < tl)
            acc[r] = __dadd_rn(acc[r], __dmul_rn(sc[ph[r] * tl + i0 + u], DT_<DT>::load(&vr[u][r])));
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (ph[r] >= 0) DT_<DT>::store((T*)out.addr + (h0 + ph[r]) * out.strides[0] + (int64_t)pj[r] * out.strides[1], acc[r]);
    group_sync(c);
  }
}

__device__ __noinline__ int op_sdpa(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 3) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& q = t->views[1];
  const gpuos_view& kk = t->views[2];
  const gpuos_view& vv = t->views[3];
  if (!is_float_dt(out.dtype)) return GPUOS_DTYPE_MISMATCH;
  if (q.dtype != out.dtype || kk.dtype != out.dtype || vv.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (q.rank != 2 || kk.rank != 3 || vv.rank != 3) return GPUOS_SHAPE_MISMATCH;
  const int h = q.extents[0], d = q.extents[1], tl = kk.extents[1];
  if (kk.extents[0] != h || kk.extents[2] != d || !same_shape(vv, kk)) return GPUOS_SHAPE_MISMATCH;
  if (!same_shape(out, q)) return GPUOS_SHAPE_MISMATCH;
  if (tl == 0) return GPUOS_EMPTY_AXIS;
  const double scale = (t->n_scalars > 0 && t->scalars[0] > 0.0) ? t->scalars[0]
                                                                  : __ddiv_rn(1.0, __dsqrt_rn((double)d));
  int bc;
  if ((bc = bind_code(q)) || (bc = bind_code(kk)) || (bc = bind_code(vv)) || (bc = bind_code(out))) return bc;
  const int dt = out.dtype;
  const bool exact = exact_products(dt);
  int64_t hlo, hhi;
  part_range(h, c->part, c->nparts, 1, &hlo, &hhi);
  const char* qp = (const char*)q.addr;
  const char* kp = (const char*)kk.addr;
  const char* vp = (const char*)vv.addr;
  // Batched heads (decode attention: a few heads, d <= 256, contexts whose
  // scores fit in scratch): see sdpa_batched.
  {
    const int hb = sdpa_heads_per_batch(c, d, tl);
    if (hb >= 1) {
      switch (dt) {
        case GPUOS_F32: sdpa_batched<GPUOS_F32>(t, c, hb, hlo, hhi, scale); break;
        case GPUOS_F64: sdpa_batched<GPUOS_F64>(t, c, hb, hlo, hhi, scale); break;
        case GPUOS_F16: sdpa_batched<GPUOS_F16>(t, c, hb, hlo, hhi, scale); break;
        default: sdpa_batched<GPUOS_BF16>(t, c, hb, hlo, hhi, scale); break;
      }
      return GPUOS_OK;
    }
  }
  double* red = (double*)c->smem;           // 32 doubles
  double* sc = red + 32;                    // score chunk
  const int cap = (c->smem_bytes - 32 * 8) / 8;
  const int chunk = cap < tl ? cap : tl;
  const bool single = chunk >= tl;
  for (int64_t head = hlo; head < hhi; ++head) {
    const int64_t qb = head * q.strides[0], kb = head * kk.strides[0], vb = head * vv.strides[0];
    auto score = [&](int i) {
      double dot = 0.0;
      for (int j = 0; j < d; ++j)
        dot = mac(dot, load_any(dt, qp, qb + (int64_t)j * q.strides[1]),
                  load_any(dt, kp, kb + (int64_t)i * kk.strides[1] + (int64_t)j * kk.strides[2]), exact);
      return __dmul_rn(scale, dot);
    };
    // pass 1: max score
    double mx = -INFINITY;
    for (int i = c->tid; i < tl; i += c->nthreads) {
      const double s = score(i);
      if (single) sc[i] = s;
      mx = nan_skip_max(mx, s);
    }
    {
      for (int o = 16; o > 0; o >>= 1) mx = nan_skip_max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((c->tid & 31) == 0) red[c->tid >> 5] = mx;
      group_sync(c);
      mx = -INFINITY;
      for (int w = 0; w < (c->nthreads >> 5); ++w) mx = nan_skip_max(mx, red[w]);
      group_sync(c);
    }
    // pass 2: denominator
    double s = 0.0;
    for (int i = c->tid; i < tl; i += c->nthreads) {
      const double e = exp(__dsub_rn(single ? sc[i] : score(i), mx));
      if (single) sc[i] = e;
      s += e;
    }
    const double denom = group_sum(s, c, red);
    // pass 3: out[j] = sum_i (e_i / denom) * v[i][j], ascending i
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i0 = 0; i0 < tl; i0 += chunk) {
      const int i1 = (i0 + chunk) < tl ? (i0 + chunk) : tl;
      if (!single) {
        for (int i = i0 + c->tid; i < i1; i += c->nthreads) sc[i - i0] = exp(__dsub_rn(score(i), mx));
        group_sync(c);
      }
      for (int r = 0; r < 4; ++r) {
        const int j = c->tid + r * c->nthreads;
        if (j >= d) break;
        double a = acc[r];
        for (int i = i0; i < i1; ++i) {
          const double w = __ddiv_rn(sc[i - (single ? 0 : i0)], denom);
          a = __dadd_rn(a, __dmul_rn(w, load_any(dt, vp, vb + (int64_t)i * vv.strides[1] + (int64_t)j * vv.strides[2])));
        }
        acc[r] = a;
      }
      group_sync(c);
    }
    for (int r = 0; r < 4; ++r) {
      const int j = c->tid + r * c->nthreads;
      if (j >= d) break;
      store_any(dt, (char*)out.addr, head * out.strides[0] + (int64_t)j * out.strides[1], acc[r]);
    }
    if (d > 4 * c->nthreads) {
      // very wide heads: remaining columns, recomputing weights from scores
      for (int j = c->tid + 4 * c->nthreads; j < d; j += c->nthreads) {
        double a = 0.0;
        for (int i = 0; i < tl; ++i) {
          const double e = single ? sc[i] : exp(__dsub_rn(score(i), mx));
          a = __dadd_rn(a, __dmul_rn(__ddiv_rn(e, denom),
                                     load_any(dt, vp, vb + (int64_t)i * vv.strides[1] + (int64_t)j * vv.strides[2])));
        }
        store_any(dt, (char*)out.addr, head * out.strides[0] + (int64_t)j * out.strides[1], a);
      }
    }
    group_sync(c);
  }
  return GPUOS_OK;
}

// ---- rope: x (t,d), positions (t) -> out (t,d) ----
__device__ __noinline__ int op_rope(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 2) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& x = t->views[1];
  const gpuos_view& pos = t->views[2];
  if (!is_float_dt(out.dtype)) return GPUOS_DTYPE_MISMATCH;
  if (x.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (x.rank != 2 || pos.rank != 1) return GPUOS_SHAPE_MISMATCH;
  if (!same_shape(out, x)) return GPUOS_SHAPE_MISMATCH;
  const int tl = x.extents[0], d = x.extents[1];
  if (pos.extents[0] != tl) return GPUOS_SHAPE_MISMATCH;
  if (d % 2 != 0) return GPUOS_ODD_DIM;
  const double base = (t->n_scalars > 0 && t->scalars[0] > 0.0) ? t->scalars[0] : 10000.0;
  int bc;
  if ((bc = bind_code(x)) || (bc = bind_code(pos)) || (bc = bind_code(out))) return bc;
  const int dt = out.dtype;
  const int half = d / 2;
  int64_t lo, hi;
  part_range((int64_t)tl * half, c->part, c->nparts, 1, &lo, &hi);
  for (int64_t e = lo + c->tid; e < hi; e += c->nthreads) {
    const int64_t r = e / half, i = e % half;
    const double p = load_any(pos.dtype, (const char*)pos.addr, r * pos.strides[0]);
    const double ex = __ddiv_rn(__dmul_rn(-2.0, (double)i), (double)d);
    const double theta = __dmul_rn(p, pow(base, ex));
    double sn, cs;
    sincos(theta, &sn, &cs);
    const int64_t xb = r * x.strides[0], ob = r * out.strides[0];
    const double x0 = load_any(dt, (const char*)x.addr, xb + (2 * i) * x.strides[1]);
    const double x1 = load_any(dt, (const char*)x.addr, xb + (2 * i + 1) * x.strides[1]);
    store_any(dt, (char*)out.addr, ob + (2 * i) * out.strides[1], __dsub_rn(__dmul_rn(x0, cs), __dmul_rn(x1, sn)));
    store_any(dt, (char*)out.addr, ob + (2 * i + 1) * out.strides[1], __dadd_rn(__dmul_rn(x0, sn), __dmul_rn(x1, cs)));
  }
  return GPUOS_OK;
}

}  // namespace gdev
