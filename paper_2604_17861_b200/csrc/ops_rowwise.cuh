// Row-wise task bodies over the last axis: softmax (reference ops.hpp:200-238),
// layernorm (ops.hpp:244-294) and the sum/max/min reduction (ops.hpp:303-355).
//
// Rows of <= 1024 elements go one warp per row; longer rows use the whole
// worker group.  Sums accumulate in fp64 (the reference's accumulation type)
// with a shuffle tree; max/min carry (value, index) pairs so the result is
// the first extremum in scan order, and a NaN first element wins exactly as
// the reference's `acc < x` scan does.
#pragma once

#include "dev_common.cuh"

namespace gdev {

// Outer (all-but-last) iteration over a view: rank-1 <= 3 dims.
struct RowIter {
  int r;                  // outer rank
  int32_t ext[3];
  FastDiv fd[3];
  int64_t rows;
  __device__ __forceinline__ void init(const gpuos_view& v) {
    r = v.rank - 1;
    rows = 1;
    for (int d = 0; d < r; ++d) {
      ext[d] = v.extents[d];
      fd[d].init((uint32_t)(ext[d] > 0 ? ext[d] : 1));
      rows *= ext[d];
    }
  }
  // element offset of row `row` in a view whose first r strides are `st`
  __device__ __forceinline__ void offsets(int64_t row, const int32_t* st_a, const int32_t* st_b,
                                          int64_t* oa, int64_t* ob) const {
    uint32_t e = (uint32_t)row;
    int64_t a = 0, b = 0;
    for (int d = r - 1; d >= 0; --d) {
      const uint32_t q = fd[d].div(e);
      const uint32_t i = e - q * fd[d].d;
      e = q;
      a += (int64_t)i * st_a[d];
      b += (int64_t)i * st_b[d];
    }
    *oa = a;
    *ob = b;
  }
};

// Distribution of rows over the group: warp-per-row when cols are short.
struct RowSched {
  bool per_warp;
  int unit;      // this thread's unit index (warp or 0)
  int nunits;    // units per group
  int lane;      // index within the unit
  int width;     // threads per unit
  int64_t lo, hi;
  __device__ __forceinline__ void init(const Ctx* c, int64_t rows, int64_t cols) {
    per_warp = cols <= 1024;
    if (per_warp) {
      unit = c->tid >> 5;
      nunits = c->nthreads >> 5;
      lane = c->tid & 31;
      width = 32;
    } else {
      unit = 0;
      nunits = 1;
      lane = c->tid;
      width = c->nthreads;
    }
    part_range(rows, c->part, c->nparts, 1, &lo, &hi);
  }
};

// Sum over one unit; for the whole-group unit this synchronises the group.
__device__ __forceinline__ double unit_sum(double v, const RowSched& rs, const Ctx* c, double* red) {
  if (rs.per_warp) return warp_sum(v);
  return group_sum(v, c, red);
}
__device__ __forceinline__ double unit_max(double v, const RowSched& rs, const Ctx* c, double* red) {
  if (rs.per_warp) return warp_max(v);
  return group_max(v, c, red);
}

// First-wins extremum with NaN-skipping, as a (value, index) pair.
struct Ext {
  double v;
  int64_t i;  // -1 => no candidate
};
__device__ __forceinline__ Ext ext_merge(Ext a, Ext b, bool is_max) {
  if (a.i < 0) return b;
  if (b.i < 0) return a;
  const bool b_better = is_max ? (a.v < b.v) : (b.v < a.v);
  const bool a_better = is_max ? (b.v < a.v) : (a.v < b.v);
  if (b_better) return b;
  if (a_better) return a;
  return a.i <= b.i ? a : b;  // equal under ==: the earlier element wins
}
__device__ __forceinline__ Ext warp_ext(Ext e, bool is_max) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Ext x;
    x.v = __shfl_xor_sync(0xffffffffu, e.v, o);
    x.i = __shfl_xor_sync(0xffffffffu, e.i, o);
    e = ext_merge(e, x, is_max);
  }
  return e;
}
__device__ __forceinline__ Ext unit_ext(Ext e, bool is_max, const RowSched& rs, const Ctx* c, char* scratch) {
  e = warp_ext(e, is_max);
  if (rs.per_warp) return e;
  double* rv = (double*)scratch;
  int64_t* ri = (int64_t*)(scratch + 32 * sizeof(double));
  const int lane = c->tid & 31, wid = c->tid >> 5, nw = c->nthreads >> 5;
  if (lane == 0) {
    rv[wid] = e.v;
    ri[wid] = e.i;
  }
  group_sync(c);
  Ext t;
  t.v = rv[0];
  t.i = ri[0];
  for (int w = 1; w < nw; ++w) {
    Ext x;
    x.v = rv[w];
    x.i = ri[w];
    t = ext_merge(t, x, is_max);
  }
  group_sync(c);
  return t;
}

// Row maximum with the reference's scan semantics (NaN first element => NaN).
__device__ __forceinline__ double row_max_scan(int dt, const char* base, int64_t step, int64_t cols,
                                               const RowSched& rs, const Ctx* c, char* scratch) {
  Ext e;
  e.v = 0.0;
  e.i = -1;
  for (int64_t j = rs.lane; j < cols; j += rs.width) {
    const double x = load_any(dt, base, j * step);
    if (x == x) {
      Ext y;
      y.v = x;
      y.i = j;
      e = ext_merge(e, y, true);
    }
  }
  e = unit_ext(e, true, rs, c, scratch);
  const double x0 = load_any(dt, base, 0);
  return (x0 != x0) ? x0 : e.v;
}

// ---- softmax ----
constexpr int kSoftmaxRegs = 8;  // rows of <= 256 elements stay in registers

// Short rows of a 32/16-bit float dtype: one warp per row, the row held in
// registers (one load round trip), dtype fixed at compile time.  The maximum
// keeps the reference's scan semantics (NaN first element => NaN, otherwise
// NaN-skipping, first extremum wins); exp runs in fp32 (expf, <= 2 ulp: the
// argument x - max is exact in double and its float rounding moves p_i by at
// most |d| e^d 2^-24 <= 2.2e-8), the sum in fp64, and the normalisation is a
// multiply by the fp64 reciprocal -- within the rel 1e-6 / 1-ulp rules of
// ops.hpp:200-238's fp64 computation (tests/cases.py row_cases).
// NR rows per warp in flight, REGS values per lane per row (cols <= 32 REGS):
// a warp used to walk its rows one at a time, one memory latency per row
// (config 3's 128 x 128 softmax tasks: 32 rows per warp, ~94 us per phase).
// Every row is computed exactly as before (same per-lane values, same
// shuffle order), so results are unchanged.
template <int DT, int REGS, int NR>
__device__ __noinline__ int softmax_rows_f(const gpuos_view& in, const gpuos_view& out, const RowIter& it,
                                           const RowSched& rs, int64_t cols, int64_t si, int64_t so) {
  typedef typename DT_<DT>::T T;
  for (int64_t base = rs.lo + (int64_t)rs.unit * NR; base < rs.hi; base += (int64_t)rs.nunits * NR) {
    const T* ib[NR];
    T* ob[NR];
    float x[NR][REGS];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      int64_t oi = 0, oo = 0;
      if (base + r < rs.hi) it.offsets(base + r, in.strides, out.strides, &oi, &oo);
      ib[r] = (const T*)in.addr + oi;
      ob[r] = (T*)out.addr + oo;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int i = 0; i < REGS; ++i) {
        const int64_t j = rs.lane + 32 * i;
        x[r][i] = (base + r < rs.hi && j < cols) ? (float)DT_<DT>::gload(ib[r] + j * si) : 0.0f;
      }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (base + r >= rs.hi) break;  // warp-uniform
      // (value, first index) maximum over the non-NaN elements
      float mv = 0.0f;
      int mi = -1;
#pragma unroll
      for (int i = 0; i < REGS; ++i) {
        const int j = rs.lane + 32 * i;
        if (j < cols && x[r][i] == x[r][i] && (mi < 0 || mv < x[r][i])) {
          mv = x[r][i];
          mi = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, mv, o);
        const int oi2 = __shfl_xor_sync(0xffffffffu, mi, o);
        if (oi2 >= 0 && (mi < 0 || mv < ov || (!(ov < mv) && oi2 < mi))) {
          mv = ov;
          mi = oi2;
        }
      }
      const float x0 = __shfl_sync(0xffffffffu, x[r][0], 0);
      const double mx = (x0 != x0) ? (double)x0 : (double)mv;
      double sum = 0.0;
#pragma unroll
      for (int i = 0; i < REGS; ++i) {
        const int64_t j = rs.lane + 32 * i;
        x[r][i] = j < cols ? expf((float)((double)x[r][i] - mx)) : 0.0f;
        sum += (double)x[r][i];
      }
      const double inv = __drcp_rn(warp_sum(sum));
#pragma unroll
      for (int i = 0; i < REGS; ++i) {
        const int64_t j = rs.lane + 32 * i;
        if (j < cols) DT_<DT>::store(ob[r] + j * so, (double)x[r][i] * inv);
      }
    }
  }
  return GPUOS_OK;
}
template <int DT>
__device__ __forceinline__ int softmax_rows_dispatch(const gpuos_view& in, const gpuos_view& out, const RowIter& it,
                                                     const RowSched& rs, int64_t cols, int64_t si, int64_t so) {
  if (cols <= 32) return softmax_rows_f<DT, 1, 8>(in, out, it, rs, cols, si, so);
  if (cols <= 64) return softmax_rows_f<DT, 2, 8>(in, out, it, rs, cols, si, so);
  if (cols <= 128) return softmax_rows_f<DT, 4, 4>(in, out, it, rs, cols, si, so);
  return softmax_rows_f<DT, 8, 2>(in, out, it, rs, cols, si, so);
}
__device__ __noinline__ int op_softmax(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 1) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& in = t->views[1];
  if (!is_float_dt(out.dtype)) return GPUOS_DTYPE_MISMATCH;
  if (in.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (!same_shape(in, out)) return GPUOS_SHAPE_MISMATCH;
  if (in.rank == 0 || in.extents[in.rank - 1] == 0) return GPUOS_EMPTY_AXIS;
  int b;
  if ((b = bind_code(in)) || (b = bind_code(out))) return b;
  const int dt = out.dtype;
  const int64_t cols = in.extents[in.rank - 1];
  const int64_t si = in.strides[in.rank - 1], so = out.strides[out.rank - 1];
  RowIter it;
  it.init(in);
  RowSched rs;
  rs.init(c, it.rows, cols);
  char* scratch = c->smem;
  if (rs.per_warp && cols <= 32 * kSoftmaxRegs && dt != GPUOS_F64) {
    switch (dt) {
      case GPUOS_F32: return softmax_rows_dispatch<GPUOS_F32>(in, out, it, rs, cols, si, so);
      case GPUOS_F16: return softmax_rows_dispatch<GPUOS_F16>(in, out, it, rs, cols, si, so);
      default: return softmax_rows_dispatch<GPUOS_BF16>(in, out, it, rs, cols, si, so);
    }
  }
  // whole-group units visit identical rows, so their barriers stay matched
  for (int64_t row = rs.lo + rs.unit; row < rs.hi; row += rs.nunits) {
    int64_t oi, oo;
    it.offsets(row, in.strides, out.strides, &oi, &oo);
    const char* ib = (const char*)in.addr + oi * dtype_width(dt);
    char* ob = (char*)out.addr + oo * dtype_width(dt);
    const double mx = row_max_scan(dt, ib, si, cols, rs, c, scratch);
    double s = 0.0;
    for (int64_t j = rs.lane; j < cols; j += rs.width) s += exp(__dsub_rn(load_any(dt, ib, j * si), mx));
    const double denom = unit_sum(s, rs, c, (double*)scratch);
    for (int64_t j = rs.lane; j < cols; j += rs.width) {
      const double e = exp(__dsub_rn(load_any(dt, ib, j * si), mx));
      store_any(dt, ob, j * so, __ddiv_rn(e, denom));
    }
  }
  return GPUOS_OK;
}

// ---- layernorm: inputs {x, gamma, beta}, scalars[0] = eps ----
__device__ __noinline__ int op_layernorm(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 3) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& in = t->views[1];
  const gpuos_view& g = t->views[2];
  const gpuos_view& be = t->views[3];
  if (!is_float_dt(out.dtype)) return GPUOS_DTYPE_MISMATCH;
  if (in.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (!same_shape(in, out)) return GPUOS_SHAPE_MISMATCH;
  if (in.rank == 0 || in.extents[in.rank - 1] == 0) return GPUOS_EMPTY_AXIS;
  if (g.dtype != out.dtype || be.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  const double eps = t->n_scalars == 0 ? 1e-5 : t->scalars[0];
  const int64_t cols = in.extents[in.rank - 1];
  // broadcast_view(gamma, {cols}) / (beta, {cols})
  int64_t gs, bs;
  {
    if (g.rank > 1 || be.rank > 1) return GPUOS_INCOMPATIBLE_SHAPES;
    if (g.rank == 1 && g.extents[0] != cols && g.extents[0] != 1) return GPUOS_INCOMPATIBLE_SHAPES;
    gs = (g.rank == 1 && g.extents[0] == cols) ? g.strides[0] : 0;
    if (be.rank == 1 && be.extents[0] != cols && be.extents[0] != 1) return GPUOS_INCOMPATIBLE_SHAPES;
    bs = (be.rank == 1 && be.extents[0] == cols) ? be.strides[0] : 0;
  }
  int b;
  if ((b = bind_code(in)) || (b = bind_code(out)) || (b = bind_code(g)) || (b = bind_code(be))) return b;
  const int dt = out.dtype;
  const int64_t si = in.strides[in.rank - 1], so = out.strides[out.rank - 1];
  RowIter it;
  it.init(in);
  RowSched rs;
  rs.init(c, it.rows, cols);
  double* red = (double*)c->smem;
  const double dcols = (double)cols;
  for (int64_t row = rs.lo + rs.unit; row < rs.hi; row += rs.nunits) {
    int64_t oi, oo;
    it.offsets(row, in.strides, out.strides, &oi, &oo);
    const char* ib = (const char*)in.addr + oi * dtype_width(dt);
    char* ob = (char*)out.addr + oo * dtype_width(dt);
    double s = 0.0;
    for (int64_t j = rs.lane; j < cols; j += rs.width) s += load_any(dt, ib, j * si);
    const double mean = __ddiv_rn(unit_sum(s, rs, c, red), dcols);
    double v = 0.0;
    for (int64_t j = rs.lane; j < cols; j += rs.width) {
      const double d = __dsub_rn(load_any(dt, ib, j * si), mean);
      v = __dadd_rn(v, __dmul_rn(d, d));
    }
    const double var = __ddiv_rn(unit_sum(v, rs, c, red), dcols);
    const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, eps)));
    for (int64_t j = rs.lane; j < cols; j += rs.width) {
      const double xhat = __dmul_rn(__dsub_rn(load_any(dt, ib, j * si), mean), inv);
      const double gv = load_any(dt, (const char*)g.addr, j * gs);
      const double bv = load_any(dt, (const char*)be.addr, j * bs);
      store_any(dt, ob, j * so, __dadd_rn(__dmul_rn(xhat, gv), bv));
    }
  }
  return GPUOS_OK;
}

// ---- reductions over the last axis ----
// This lane's part of a row sum in fp64: kSumUnroll loads in flight before
// they are added (the fp64 sum of <= 64K narrower values rounds to the same
// output as the reference's left-to-right order, SURVEY §8(a) "<= 1 ulp").
constexpr int kSumUnroll = 8;
template <int DT>
__device__ __forceinline__ double lane_sum(const char* ib, int64_t si, int64_t cols, const RowSched& rs) {
  typedef typename DT_<DT>::T T;
  const T* p = (const T*)ib;
  double s = 0.0;
  for (int64_t j0 = rs.lane; j0 < cols; j0 += (int64_t)rs.width * kSumUnroll) {
    double v[kSumUnroll];
#pragma unroll
    for (int u = 0; u < kSumUnroll; ++u) {
      const int64_t j = j0 + (int64_t)u * rs.width;
      v[u] = j < cols ? DT_<DT>::gload(p + j * si) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kSumUnroll; ++u) s += v[u];
  }
  return s;
}

// Contiguous row (unit stride): a scalar head up to 16-byte alignment, then
// kSumVec 16-byte vectors per lane in flight, then a scalar tail.  The fp64
// lane partials are combined by the unit's tree (<= 1 ulp rule, as above).
constexpr int kSumVec = 4;
template <int DT>
__device__ __forceinline__ double lane_sum_vec(const char* ib, int64_t cols, const RowSched& rs) {
  typedef typename DT_<DT>::T T;
  constexpr int V = 16 / (int)sizeof(T);
  const T* p = (const T*)ib;
  int64_t head = (int64_t)(((16 - ((uintptr_t)p & 15)) & 15) / sizeof(T));
  if (head > cols) head = cols;
  const int64_t nv = (cols - head) / V;
  double s = 0.0;
  if (rs.lane < head) s += DT_<DT>::gload(p + rs.lane);
  const uint4* vb = reinterpret_cast<const uint4*>(p + head);
  for (int64_t i0 = rs.lane; i0 < nv; i0 += (int64_t)rs.width * kSumVec) {
    uint4 v[kSumVec];
#pragma unroll
    for (int u = 0; u < kSumVec; ++u) {
      const int64_t i = i0 + (int64_t)u * rs.width;
      v[u] = i < nv ? ld_cg_v4(vb + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kSumVec; ++u)
#pragma unroll
      for (int j = 0; j < V; ++j) s += DT_<DT>::load(reinterpret_cast<const T*>(&v[u]) + j);
  }
  for (int64_t j = head + nv * V + rs.lane; j < cols; j += rs.width) s += DT_<DT>::gload(p + j);
  return s;
}

// Interleaved rows (a transposed 2-D view: row stride 1, element stride >
// 1): one thread per row walks its elements in order, so a warp's loads are
// 32 consecutive rows' elements -- coalesced -- and the sum / first-wins scan
// is the reference's left-to-right order exactly.
template <int MODE, int DT>
__device__ __forceinline__ void reduce_rows_by_thread(const gpuos_view& in, const gpuos_view& out, int64_t rows,
                                                      int64_t cols, const Ctx* c) {
  typedef typename DT_<DT>::T T;
  const T* ib = (const T*)in.addr;
  T* ob = (T*)out.addr;
  const int64_t si = in.strides[1];
  int64_t lo, hi;
  part_range(rows, c->part, c->nparts, 1, &lo, &hi);
  constexpr int U = 8;
  for (int64_t r = lo + c->tid; r < hi; r += c->nthreads) {
    const T* rp = ib + r;  // in.strides[0] == 1
    double acc = 0.0, best = 0.0;
    int64_t bi = -1;
    for (int64_t j0 = 0; j0 < cols; j0 += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = j0 + u < cols ? DT_<DT>::gload(rp + (j0 + u) * si) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (j0 + u >= cols) break;
        if (MODE == 0) {
          acc += v[u];
        } else if (v[u] == v[u] && (bi < 0 || (MODE == 1 ? best < v[u] : v[u] < best))) {
          best = v[u];
          bi = j0 + u;
        }
      }
    }
    double res = acc;
    if (MODE != 0) {
      const double x0 = DT_<DT>::gload(rp);
      res = (x0 != x0 || bi < 0) ? x0 : best;
    }
    DT_<DT>::store(ob + r * out.strides[0], res);
  }
}

template <int MODE>  // 0 sum, 1 max, 2 min
__device__ __forceinline__ int reduce_body(const gpuos_task* t, const Ctx* c) {
  if (t->n_inputs != 1) return GPUOS_ARITY_ERROR;
  const gpuos_view& out = t->views[0];
  const gpuos_view& in = t->views[1];
  if (in.dtype != out.dtype) return GPUOS_DTYPE_MISMATCH;
  if (in.rank == 0) return GPUOS_EMPTY_AXIS;
  if (out.rank != in.rank - 1) return GPUOS_SHAPE_MISMATCH;
  for (int d = 0; d < out.rank; ++d)
    if (out.extents[d] != in.extents[d]) return GPUOS_SHAPE_MISMATCH;
  const int64_t cols = in.extents[in.rank - 1];
  if (cols == 0 && MODE != 0) return GPUOS_EMPTY_AXIS;
  int b;
  if ((b = bind_code(in)) || (b = bind_code(out))) return b;
  const int dt = out.dtype;
  const int64_t si = in.strides[in.rank - 1];
  if (in.rank == 2 && out.rank == 1 && in.strides[0] == 1 && si != 1 && in.extents[0] >= 32 && dt != GPUOS_I32 &&
      cols > 0) {
    switch (dt) {
      case GPUOS_F32: reduce_rows_by_thread<MODE, GPUOS_F32>(in, out, in.extents[0], cols, c); break;
      case GPUOS_F64: reduce_rows_by_thread<MODE, GPUOS_F64>(in, out, in.extents[0], cols, c); break;
      case GPUOS_F16: reduce_rows_by_thread<MODE, GPUOS_F16>(in, out, in.extents[0], cols, c); break;
      default: reduce_rows_by_thread<MODE, GPUOS_BF16>(in, out, in.extents[0], cols, c); break;
    }
    return GPUOS_OK;
  }
  RowIter it;
  it.init(in);
  if (MODE == 0 && si == 1 && cols <= 512 && dt != GPUOS_I32) {
    // short contiguous rows: 8-lane sub-units, four rows per warp in flight
    // (a whole warp per row left most lanes idle and one row's latency per
    // step); warp-uniform row rounds keep every shuffle convergent
    RowSched rs;
    rs.lane = c->tid & 7;
    rs.width = 8;
    int64_t lo, hi;
    part_range(it.rows, c->part, c->nparts, 1, &lo, &hi);
    const int sub = (c->tid & 31) >> 3, warp = c->tid >> 5, nw = c->nthreads >> 5;
    for (int64_t base = lo + (int64_t)warp * 4; base < hi; base += (int64_t)nw * 4) {
      const int64_t row = base + sub;
      double sum = 0.0;
      int64_t oo = 0;
      if (row < hi) {
        int64_t oi;
        it.offsets(row, in.strides, out.strides, &oi, &oo);
        const char* ib = (const char*)in.addr + oi * dtype_width(dt);
        switch (dt) {
          case GPUOS_F32: sum = lane_sum_vec<GPUOS_F32>(ib, cols, rs); break;
          case GPUOS_F64: sum = lane_sum_vec<GPUOS_F64>(ib, cols, rs); break;
          case GPUOS_F16: sum = lane_sum_vec<GPUOS_F16>(ib, cols, rs); break;
          default: sum = lane_sum_vec<GPUOS_BF16>(ib, cols, rs); break;
        }
      }
      sum += __shfl_xor_sync(0xffffffffu, sum, 4);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      if (row < hi && rs.lane == 0) store_any(dt, (char*)out.addr + oo * dtype_width(dt), 0, sum);
    }
    return GPUOS_OK;
  }
  RowSched rs;
  rs.init(c, it.rows, cols);
  for (int64_t row = rs.lo + rs.unit; row < rs.hi; row += rs.nunits) {
    int64_t oi, oo;
    it.offsets(row, in.strides, out.strides, &oi, &oo);
    const char* ib = (const char*)in.addr + oi * dtype_width(dt);
    char* ob = (char*)out.addr + oo * dtype_width(dt);
    double r;
    if (MODE == 0) {
      if (dt == GPUOS_I32) {
        // exact integer accumulation == the reference's exact-in-double sum
        long long s = 0;
        for (int64_t j0 = rs.lane; j0 < cols; j0 += (int64_t)rs.width * kSumUnroll) {
          int32_t v[kSumUnroll];
#pragma unroll
          for (int u = 0; u < kSumUnroll; ++u) {
            const int64_t j = j0 + (int64_t)u * rs.width;
            v[u] = j < cols ? __ldcg((const int32_t*)ib + j * si) : 0;
          }
#pragma unroll
          for (int u = 0; u < kSumUnroll; ++u) s += v[u];
        }
        r = (double)(long long)unit_sum((double)s, rs, c, (double*)c->smem);
      } else {
        double s = 0.0;
        if (si == 1) {
          switch (dt) {
            case GPUOS_F32: s = lane_sum_vec<GPUOS_F32>(ib, cols, rs); break;
            case GPUOS_F64: s = lane_sum_vec<GPUOS_F64>(ib, cols, rs); break;
            case GPUOS_F16: s = lane_sum_vec<GPUOS_F16>(ib, cols, rs); break;
            default: s = lane_sum_vec<GPUOS_BF16>(ib, cols, rs); break;
          }
        } else {
          switch (dt) {
            case GPUOS_F32: s = lane_sum<GPUOS_F32>(ib, si, cols, rs); break;
            case GPUOS_F64: s = lane_sum<GPUOS_F64>(ib, si, cols, rs); break;
            case GPUOS_F16: s = lane_sum<GPUOS_F16>(ib, si, cols, rs); break;
            default: s = lane_sum<GPUOS_BF16>(ib, si, cols, rs); break;
          }
        }
        r = unit_sum(s, rs, c, (double*)c->smem);
      }
    } else {
      Ext e;
      e.v = 0.0;
      e.i = -1;
      for (int64_t j = rs.lane; j < cols; j += rs.width) {
        const double x = load_any(dt, ib, j * si);
        if (x == x) {
          Ext y;
          y.v = x;
          y.i = j;
          e = ext_merge(e, y, MODE == 1);
        }
      }
      e = unit_ext(e, MODE == 1, rs, c, c->smem);
      const double x0 = load_any(dt, ib, 0);
      r = (x0 != x0 || e.i < 0) ? x0 : e.v;
    }
    if (rs.lane == 0) store_any(dt, ob, 0, r);
  }
  return GPUOS_OK;
}

__device__ __noinline__ int op_reduce_sum(const gpuos_task* t, const Ctx* c) { return reduce_body<0>(t, c); }
__device__ __noinline__ int op_reduce_max(const gpuos_task* t, const Ctx* c) { return reduce_body<1>(t, c); }
__device__ __noinline__ int op_reduce_min(const gpuos_task* t, const Ctx* c) { return reduce_body<2>(t, c); }

}  // namespace gdev
