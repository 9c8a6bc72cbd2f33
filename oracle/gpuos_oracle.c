/*
 * gpuos_oracle.c — CPU restatement of the reference task bodies.
 * TEST INFRASTRUCTURE ONLY (see gpuos_oracle.h): used by tests/ and
 * __graft_entry__.smoke() as the parity checker, never by the product.
 * Built with -ffp-contract=off like the reference (CMakeLists.txt:11-15).
 */
#include "gpuos_oracle.h"

#include <math.h>
#include <stdint.h>
#include <string.h>

enum {
  E_OK = 0, E_INCOMPATIBLE = 1, E_OOB = 2, E_INVALID_BUFFER = 3, E_ARITY = 13, E_VERIFY = 14, E_EMPTY_AXIS = 15,
  E_DTYPE = 16, E_SHAPE = 17, E_TOO_LARGE = 18, E_ODD_DIM = 19, E_CACHE_FULL = 20
};

/* ---- dtype conversions: tensor.hpp:259-285 ---- */

int32_t orc_narrow_i32(double v) {
  /* static_cast<int32_t>(double) as x86 cvttsd2si: truncate, INT32_MIN when
     out of range or NaN */
  if (v > -2147483649.0 && v < 2147483648.0) return (int32_t)v;
  return INT32_MIN;
}

/* Round-to-nearest-even of an exact double to a binary16/bfloat16 pattern:
   a single rounding, the rule BoundView::store applies for F32 (new dtypes,
   labelled restatement). */
static uint16_t narrow_bits(double x, int frac, int emin, int emax) {
  const uint16_t sign = signbit(x) ? 0x8000u : 0u;
  const uint16_t exp_all = (uint16_t)((2 * emax + 1) << frac);
  if (isnan(x)) return (uint16_t)(sign | exp_all | (1u << (frac - 1)));
  const double a = fabs(x);
  if (a >= ldexp(2.0 - ldexp(1.0, -frac - 1), emax)) return (uint16_t)(sign | exp_all);
  if (a < ldexp(1.0, emin)) return (uint16_t)(sign | (uint16_t)nearbyint(ldexp(a, frac - emin)));
  int e2;
  frexp(a, &e2);
  int e = e2 - 1;
  double m = nearbyint(ldexp(a, frac - e));
  if (m >= ldexp(1.0, frac + 1)) {
    m = ldexp(1.0, frac);
    ++e;
  }
  if (e > emax) return (uint16_t)(sign | exp_all);
  return (uint16_t)(sign | ((uint32_t)(e + emax) << frac) | ((uint32_t)m - (1u << frac)));
}
static double widen_bits(uint16_t b, int frac, int emin, int emax) {
  const uint32_t e = (b & 0x7fffu) >> frac, f = b & ((1u << frac) - 1);
  double v;
  if (e == 0) v = ldexp((double)f, emin - frac);
  else if (e == (uint32_t)(2 * emax + 1)) v = f ? NAN : INFINITY;
  else v = ldexp((double)(f | (1u << frac)), (int)e - emax - frac);
  return (b & 0x8000u) ? -v : v;
}
uint16_t orc_f16_bits(double v) { return narrow_bits(v, 10, -14, 15); }
uint16_t orc_bf16_bits(double v) { return narrow_bits(v, 7, -126, 127); }
double orc_f16_value(uint16_t b) { return widen_bits(b, 10, -14, 15); }
double orc_bf16_value(uint16_t b) { return widen_bits(b, 7, -126, 127); }

double orc_load(int dt, const void* base, int64_t i) {
  switch (dt) {
    case ORC_F32: return (double)((const float*)base)[i];
    case ORC_F64: return ((const double*)base)[i];
    case ORC_I32: return (double)((const int32_t*)base)[i];
    case ORC_F16: return orc_f16_value(((const uint16_t*)base)[i]);
    default: return orc_bf16_value(((const uint16_t*)base)[i]);
  }
}
void orc_store(int dt, void* base, int64_t i, double v) {
  switch (dt) {
    case ORC_F32: ((float*)base)[i] = (float)v; break;
    case ORC_F64: ((double*)base)[i] = v; break;
    case ORC_I32: ((int32_t*)base)[i] = orc_narrow_i32(v); break;
    case ORC_F16: ((uint16_t*)base)[i] = orc_f16_bits(v); break;
    default: ((uint16_t*)base)[i] = orc_bf16_bits(v); break;
  }
}
double orc_narrow(int dt, double v) {  /* narrow_to, tensor.hpp:278-285 */
  switch (dt) {
    case ORC_F32: return (double)(float)v;
    case ORC_F64: return v;
    case ORC_I32: return (double)orc_narrow_i32(v);
    case ORC_F16: return orc_f16_value(orc_f16_bits(v));
    default: return orc_bf16_value(orc_bf16_bits(v));
  }
}

/* BoundView construction checks (tensor.hpp:246-256). */
static int bind(const orc_view* v) {
  if (v->buf_dtype < 0) return E_INVALID_BUFFER;
  if (v->buf_dtype != v->dtype) return E_DTYPE;
  return E_OK;
}
static int64_t numel(const orc_view* v) {
  int64_t n = 1;
  for (int d = 0; d < v->rank; ++d) n *= v->shape[d];
  return n;
}
static int same_shape(const orc_view* a, const orc_view* b) {
  if (a->rank != b->rank) return 0;
  for (int d = 0; d < a->rank; ++d)
    if (a->shape[d] != b->shape[d]) return 0;
  return 1;
}

int orc_broadcast_shapes(const int64_t* a, int ra, const int64_t* b, int rb, int64_t* out, int* rout) {
  const int r = ra > rb ? ra : rb;  /* tensor.hpp:104-124 */
  for (int i = 0; i < r; ++i) {
    const int64_t da = i < ra ? a[ra - 1 - i] : 1, db = i < rb ? b[rb - 1 - i] : 1;
    if (da != db && da != 1 && db != 1) return E_INCOMPATIBLE;
    out[r - 1 - i] = da > db ? da : db;
  }
  *rout = r;
  return E_OK;
}

/* broadcast_view (tensor.hpp:126-147): strides of `v` expanded to target. */
static int broadcast_view(const orc_view* v, const int64_t* target, int rt, orc_view* out) {
  if (v->rank > rt) return E_INCOMPATIBLE;
  *out = *v;
  out->rank = rt;
  for (int i = 0; i < rt; ++i) {
    out->shape[i] = target[i];
    out->strides[i] = 0;
  }
  for (int i = 0; i < v->rank; ++i) {
    const int64_t dv = v->shape[v->rank - 1 - i], dt = target[rt - 1 - i];
    if (dv == dt) out->strides[rt - 1 - i] = v->strides[v->rank - 1 - i];
    else if (dv == 1) out->strides[rt - 1 - i] = 0;
    else return E_INCOMPATIBLE;
  }
  return E_OK;
}

/* Row-major odometer over a shape with per-operand offsets (IndexIterator,
   tensor.hpp:289-325). */
typedef struct {
  int rank, nops;
  int64_t shape[ORC_MAX_RANK], idx[ORC_MAX_RANK];
  int64_t off[6];
  int64_t st[6][ORC_MAX_RANK];
} odo;
static void odo_init(odo* it, const int64_t* shape, int rank, orc_view** ops, int nops) {
  it->rank = rank;
  it->nops = nops;
  for (int d = 0; d < rank; ++d) {
    it->shape[d] = shape[d];
    it->idx[d] = 0;
  }
  for (int o = 0; o < nops; ++o) {
    it->off[o] = ops[o]->offset;
    for (int d = 0; d < rank; ++d) it->st[o][d] = ops[o]->strides[d];
  }
}
static void odo_next(odo* it) {
  for (int d = it->rank - 1; d >= 0; --d) {
    ++it->idx[d];
    for (int o = 0; o < it->nops; ++o) it->off[o] += it->st[o][d];
    if (it->idx[d] < it->shape[d]) return;
    for (int o = 0; o < it->nops; ++o) it->off[o] -= it->st[o][d] * it->shape[d];
    it->idx[d] = 0;
  }
}

/* ---- elementwise (ops.hpp:79-82, 133-194) ---- */
static double gelu_scalar(double x) {
  const double c = sqrt(2.0 / 3.14159265358979323846);
  return 0.5 * x * (1.0 + tanh(c * (x + 0.044715 * x * x * x)));
}

int orc_elementwise(int op, orc_view* out, orc_view* in, int n_in) {
  const int arity = (op <= 1) ? 2 : 1;
  if (n_in != arity) return E_ARITY;
  if (op == 3 && out->dtype == ORC_I32) return E_DTYPE; /* require_float for gelu */
  for (int i = 0; i < arity; ++i)
    if (in[i].dtype != out->dtype) return E_DTYPE;
  const int64_t n = numel(out);
  if (n == 0) return E_OK;
  orc_view b[4];
  for (int i = 0; i < arity; ++i) {
    int rc = broadcast_view(&in[i], out->shape, out->rank, &b[i]);
    if (rc) return rc;
    if ((rc = bind(&in[i]))) return rc;
  }
  int rc = bind(out);
  if (rc) return rc;
  orc_view* ops[5];
  for (int i = 0; i < arity; ++i) ops[i] = &b[i];
  ops[arity] = out;
  odo it;
  odo_init(&it, out->shape, out->rank, ops, arity + 1);
  for (int64_t e = 0; e < n; ++e) {
    double v[2] = {0, 0};
    for (int i = 0; i < arity; ++i) v[i] = orc_load(b[i].dtype, b[i].base, it.off[i]);
    double r;
    switch (op) {
      case 0: r = v[0] + v[1]; break;
      case 1: r = v[0] * v[1]; break;
      case 2: r = v[0] < 0.0 ? 0.0 : v[0]; break;
      default: r = gelu_scalar(v[0]); break;
    }
    orc_store(out->dtype, out->base, it.off[arity], r);
    odo_next(&it);
  }
  return E_OK;
}

/* Outer (all-but-last) iteration shared by the row kernels. */
static void outer_view(const orc_view* v, orc_view* o) {
  *o = *v;
  o->rank = v->rank - 1;
}

/* ---- softmax (ops.hpp:200-238) ---- */
int orc_softmax(orc_view* out, orc_view* in) {
  if (out->dtype == ORC_I32) return E_DTYPE;
  if (in->dtype != out->dtype) return E_DTYPE;
  if (!same_shape(in, out)) return E_SHAPE;
  if (in->rank == 0 || in->shape[in->rank - 1] == 0) return E_EMPTY_AXIS;
  const int64_t cols = in->shape[in->rank - 1];
  const int64_t si = in->strides[in->rank - 1], so = out->strides[out->rank - 1];
  orc_view io, oo;
  outer_view(in, &io);
  outer_view(out, &oo);
  int rc;
  if ((rc = bind(in)) || (rc = bind(out))) return rc;
  orc_view* ops[2] = {&io, &oo};
  odo it;
  odo_init(&it, io.shape, io.rank, ops, 2);
  const int64_t rows = numel(&io);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t bi = it.off[0], bo = it.off[1];
    double mx = orc_load(in->dtype, in->base, bi);
    for (int64_t j = 1; j < cols; ++j) {
      const double x = orc_load(in->dtype, in->base, bi + j * si);
      if (mx < x) mx = x;
    }
    double den = 0.0;
    for (int64_t j = 0; j < cols; ++j) den += exp(orc_load(in->dtype, in->base, bi + j * si) - mx);
    for (int64_t j = 0; j < cols; ++j)
      orc_store(out->dtype, out->base, bo + j * so, exp(orc_load(in->dtype, in->base, bi + j * si) - mx) / den);
    odo_next(&it);
  }
  return E_OK;
}

/* ---- layernorm (ops.hpp:244-294) ---- */
int orc_layernorm(orc_view* out, orc_view* in, orc_view* g, orc_view* be, double eps_in, int has_eps) {
  if (out->dtype == ORC_I32) return E_DTYPE;
  if (in->dtype != out->dtype) return E_DTYPE;
  if (!same_shape(in, out)) return E_SHAPE;
  if (in->rank == 0 || in->shape[in->rank - 1] == 0) return E_EMPTY_AXIS;
  if (g->dtype != out->dtype || be->dtype != out->dtype) return E_DTYPE;
  const double eps = has_eps ? eps_in : 1e-5;
  const int64_t cols = in->shape[in->rank - 1];
  orc_view gb, bb;
  int rc;
  if ((rc = broadcast_view(g, &cols, 1, &gb))) return rc;
  if ((rc = broadcast_view(be, &cols, 1, &bb))) return rc;
  const int64_t si = in->strides[in->rank - 1], so = out->strides[out->rank - 1];
  orc_view io, oo;
  outer_view(in, &io);
  outer_view(out, &oo);
  if ((rc = bind(in)) || (rc = bind(out)) || (rc = bind(g)) || (rc = bind(be))) return rc;
  orc_view* ops[2] = {&io, &oo};
  odo it;
  odo_init(&it, io.shape, io.rank, ops, 2);
  const int64_t rows = numel(&io);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t bi = it.off[0], bo = it.off[1];
    double mean = 0.0;
    for (int64_t j = 0; j < cols; ++j) mean += orc_load(in->dtype, in->base, bi + j * si);
    mean /= (double)cols;
    double var = 0.0;
    for (int64_t j = 0; j < cols; ++j) {
      const double d = orc_load(in->dtype, in->base, bi + j * si) - mean;
      var += d * d;
    }
    var /= (double)cols;
    const double inv = 1.0 / sqrt(var + eps);
    for (int64_t j = 0; j < cols; ++j) {
      const double xh = (orc_load(in->dtype, in->base, bi + j * si) - mean) * inv;
      const double gv = orc_load(g->dtype, g->base, gb.offset + j * gb.strides[0]);
      const double bv = orc_load(be->dtype, be->base, bb.offset + j * bb.strides[0]);
      orc_store(out->dtype, out->base, bo + j * so, xh * gv + bv);
    }
    odo_next(&it);
  }
  return E_OK;
}

/* ---- reductions over the last axis (ops.hpp:303-355) ---- */
int orc_reduce(int mode, orc_view* out, orc_view* in) {
  if (in->dtype != out->dtype) return E_DTYPE;
  if (in->rank == 0) return E_EMPTY_AXIS;
  orc_view io;
  outer_view(in, &io);
  if (!same_shape(&io, out)) return E_SHAPE;
  const int64_t cols = in->shape[in->rank - 1];
  if (cols == 0 && mode != 0) return E_EMPTY_AXIS;
  const int64_t si = in->strides[in->rank - 1];
  int rc;
  if ((rc = bind(in)) || (rc = bind(out))) return rc;
  orc_view* ops[2] = {&io, out};
  odo it;
  odo_init(&it, io.shape, io.rank, ops, 2);
  const int64_t rows = numel(&io);
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t bi = it.off[0];
    double acc;
    if (mode == 0) {
      acc = 0.0;
      for (int64_t j = 0; j < cols; ++j) acc += orc_load(in->dtype, in->base, bi + j * si);
    } else {
      acc = orc_load(in->dtype, in->base, bi);
      for (int64_t j = 1; j < cols; ++j) {
        const double x = orc_load(in->dtype, in->base, bi + j * si);
        if (mode == 1 ? (acc < x) : (x < acc)) acc = x;
      }
    }
    orc_store(out->dtype, out->base, it.off[1], acc);
    odo_next(&it);
  }
  return E_OK;
}

/* ---- matmul / vecmat (ops.hpp:363-433) ---- */
int orc_matmul(orc_view* out, orc_view* a, orc_view* b, int64_t max_dim) {
  if (a->dtype != out->dtype || b->dtype != out->dtype) return E_DTYPE;
  if (a->rank != 2 || b->rank != 2 || out->rank != 2) return E_SHAPE;
  const int64_t m = a->shape[0], k = a->shape[1], n = b->shape[1];
  if (b->shape[0] != k) return E_SHAPE;
  if (out->shape[0] != m || out->shape[1] != n) return E_SHAPE;
  if (max_dim > 0 && (m > max_dim || k > max_dim || n > max_dim)) return E_TOO_LARGE;
  int rc;
  if ((rc = bind(a)) || (rc = bind(b)) || (rc = bind(out))) return rc;
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p)
        acc += orc_load(a->dtype, a->base, a->offset + i * a->strides[0] + p * a->strides[1]) *
               orc_load(b->dtype, b->base, b->offset + p * b->strides[0] + j * b->strides[1]);
      orc_store(out->dtype, out->base, out->offset + i * out->strides[0] + j * out->strides[1], acc);
    }
  return E_OK;
}

int orc_vecmat(orc_view* out, orc_view* v, orc_view* mt, int64_t max_dim) {
  if (v->dtype != out->dtype || mt->dtype != out->dtype) return E_DTYPE;
  if (v->rank != 1 || mt->rank != 2 || out->rank != 1) return E_SHAPE;
  const int64_t k = v->shape[0], n = mt->shape[1];
  if (mt->shape[0] != k || out->shape[0] != n) return E_SHAPE;
  if (max_dim > 0 && (k > max_dim || n > max_dim)) return E_TOO_LARGE;
  int rc;
  if ((rc = bind(v)) || (rc = bind(mt)) || (rc = bind(out))) return rc;
  for (int64_t j = 0; j < n; ++j) {
    double acc = 0.0;
    for (int64_t p = 0; p < k; ++p)
      acc += orc_load(v->dtype, v->base, v->offset + p * v->strides[0]) *
             orc_load(mt->dtype, mt->base, mt->offset + p * mt->strides[0] + j * mt->strides[1]);
    orc_store(out->dtype, out->base, out->offset + j * out->strides[0], acc);
  }
  return E_OK;
}

/* ---- sdpa (ops.hpp:441-498) ---- */
int orc_sdpa(orc_view* out, orc_view* q, orc_view* k, orc_view* v, double scale_in, int has_scale) {
  if (out->dtype == ORC_I32) return E_DTYPE;
  if (q->dtype != out->dtype || k->dtype != out->dtype || v->dtype != out->dtype) return E_DTYPE;
  if (q->rank != 2 || k->rank != 3 || v->rank != 3) return E_SHAPE;
  const int64_t h = q->shape[0], d = q->shape[1], t = k->shape[1];
  if (k->shape[0] != h || k->shape[2] != d || !same_shape(v, k)) return E_SHAPE;
  if (!same_shape(out, q)) return E_SHAPE;
  if (t == 0) return E_EMPTY_AXIS;
  const double scale = (has_scale && scale_in > 0.0) ? scale_in : 1.0 / sqrt((double)d);
  int rc;
  if ((rc = bind(q)) || (rc = bind(k)) || (rc = bind(v)) || (rc = bind(out))) return rc;
  double scores[65536];
  double accum[4096];
  if (t > 65536 || d > 4096) return E_TOO_LARGE;  /* oracle sizing only */
  for (int64_t hd = 0; hd < h; ++hd) {
    const int64_t qb = q->offset + hd * q->strides[0], kb = k->offset + hd * k->strides[0];
    const int64_t vb = v->offset + hd * v->strides[0], ob = out->offset + hd * out->strides[0];
    double mx = -INFINITY;
    for (int64_t i = 0; i < t; ++i) {
      double dot = 0.0;
      for (int64_t j = 0; j < d; ++j)
        dot += orc_load(q->dtype, q->base, qb + j * q->strides[1]) *
               orc_load(k->dtype, k->base, kb + i * k->strides[1] + j * k->strides[2]);
      scores[i] = scale * dot;
      if (mx < scores[i]) mx = scores[i];
    }
    double den = 0.0;
    for (int64_t i = 0; i < t; ++i) {
      scores[i] = exp(scores[i] - mx);
      den += scores[i];
    }
    for (int64_t j = 0; j < d; ++j) accum[j] = 0.0;
    for (int64_t i = 0; i < t; ++i) {
      const double w = scores[i] / den;
      for (int64_t j = 0; j < d; ++j)
        accum[j] += w * orc_load(v->dtype, v->base, vb + i * v->strides[1] + j * v->strides[2]);
    }
    for (int64_t j = 0; j < d; ++j) orc_store(out->dtype, out->base, ob + j * out->strides[1], accum[j]);
  }
  return E_OK;
}

/* ---- rope (ops.hpp:503-537) ---- */
int orc_rope(orc_view* out, orc_view* x, orc_view* pos, double base_in, int has_base) {
  if (out->dtype == ORC_I32) return E_DTYPE;
  if (x->dtype != out->dtype) return E_DTYPE;
  if (x->rank != 2 || pos->rank != 1) return E_SHAPE;
  if (!same_shape(out, x)) return E_SHAPE;
  const int64_t t = x->shape[0], d = x->shape[1];
  if (pos->shape[0] != t) return E_SHAPE;
  if (d % 2 != 0) return E_ODD_DIM;
  const double base = (has_base && base_in > 0.0) ? base_in : 10000.0;
  int rc;
  if ((rc = bind(x)) || (rc = bind(pos)) || (rc = bind(out))) return rc;
  for (int64_t r = 0; r < t; ++r) {
    const double p = orc_load(pos->dtype, pos->base, pos->offset + r * pos->strides[0]);
    const int64_t xb = x->offset + r * x->strides[0], ob = out->offset + r * out->strides[0];
    for (int64_t i = 0; i < d / 2; ++i) {
      const double theta = p * pow(base, -2.0 * (double)i / (double)d);
      const double c = cos(theta), s = sin(theta);
      const double x0 = orc_load(x->dtype, x->base, xb + (2 * i) * x->strides[1]);
      const double x1 = orc_load(x->dtype, x->base, xb + (2 * i + 1) * x->strides[1]);
      orc_store(out->dtype, out->base, ob + (2 * i) * out->strides[1], x0 * c - x1 * s);
      orc_store(out->dtype, out->base, ob + (2 * i + 1) * out->strides[1], x0 * s + x1 * c);
    }
  }
  return E_OK;
}

/* ---- kv_append (ops.hpp:544-589) ---- */
int orc_kv_append(orc_view* kc, orc_view* vc, orc_view* nk, orc_view* nv, double cursor_d) {
  if (kc->rank != 3 || vc->rank != 3 || nk->rank != 2 || nv->rank != 2) return E_SHAPE;
  const int64_t h = kc->shape[0], cap = kc->shape[1], d = kc->shape[2];
  if (!same_shape(vc, kc)) return E_SHAPE;
  if (nk->shape[0] != h || nk->shape[1] != d || nv->shape[0] != h || nv->shape[1] != d) return E_SHAPE;
  if (nk->dtype != kc->dtype || nv->dtype != vc->dtype || vc->dtype != kc->dtype) return E_DTYPE;
  const int64_t cursor = (cursor_d > -9.2e18 && cursor_d < 9.2e18) ? (int64_t)cursor_d : -1;
  if (cursor < 0 || cursor >= cap) return E_CACHE_FULL;
  int rc;
  if ((rc = bind(kc)) || (rc = bind(vc)) || (rc = bind(nk)) || (rc = bind(nv))) return rc;
  for (int64_t hd = 0; hd < h; ++hd) {
    const int64_t ko = kc->offset + hd * kc->strides[0] + cursor * kc->strides[1];
    const int64_t vo = vc->offset + hd * vc->strides[0] + cursor * vc->strides[1];
    const int64_t no = nk->offset + hd * nk->strides[0], mo = nv->offset + hd * nv->strides[0];
    for (int64_t j = 0; j < d; ++j) {
      orc_store(kc->dtype, kc->base, ko + j * kc->strides[2], orc_load(nk->dtype, nk->base, no + j * nk->strides[1]));
      orc_store(vc->dtype, vc->base, vo + j * vc->strides[2], orc_load(nv->dtype, nv->base, mo + j * nv->strides[1]));
    }
  }
  return E_OK;
}

/* ---- injected programs (bytecode.hpp:205-230 over opcompiler.hpp:70-122) ---- */
static double bmax(double a, double b) { return a < b ? b : a; } /* expr.hpp:134 */
static double bmin(double a, double b) { return b < a ? b : a; } /* expr.hpp:135 */

static double run(const orc_instr* code, int n, const double* in) {
  double st[256];
  int sp = 0;
  for (int pc = 0; pc < n; ++pc) {
    const orc_instr* c = &code[pc];
    switch (c->op) {
      case 0: st[sp++] = c->value; break;
      case 1: st[sp++] = in[c->k]; break;
      case 2: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
      case 3: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
      case 4: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
      case 5: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
      case 6: st[sp - 1] = -st[sp - 1]; break;
      case 7: st[sp - 1] = exp(st[sp - 1]); break;
      case 8: st[sp - 1] = tanh(st[sp - 1]); break;
      case 9: --sp; st[sp - 1] = bmax(st[sp - 1], st[sp]); break;
      case 10: --sp; st[sp - 1] = bmin(st[sp - 1], st[sp]); break;
      case 11: st[sp - 1] = fabs(st[sp - 1]); break;
      case 12: st[sp - 1] = sqrt(st[sp - 1]); break;
      case 13: st[sp - 1] = orc_narrow(c->k, st[sp - 1]); break;
      default: return st[--sp];
    }
  }
  return 0.0;
}

int orc_program(const orc_instr* code, int n, int arity, int dtype, orc_view* out, orc_view* in, int n_in) {
  if (n_in != arity) return E_ARITY;
  if (out->dtype != dtype) return E_DTYPE;
  const int64_t ne = numel(out);
  if (ne == 0) return E_OK;
  orc_view b[4];
  orc_view* ops[5];
  for (int i = 0; i < arity; ++i) {
    if (in[i].dtype != out->dtype) return E_DTYPE;
    int rc = broadcast_view(&in[i], out->shape, out->rank, &b[i]);
    if (rc) return rc;
    if ((rc = bind(&in[i]))) return rc;
    ops[i] = &b[i];
  }
  int rc = bind(out);
  if (rc) return rc;
  ops[arity] = out;
  odo it;
  odo_init(&it, out->shape, out->rank, ops, arity + 1);
  for (int64_t e = 0; e < ne; ++e) {
    double v[4] = {0, 0, 0, 0};
    for (int i = 0; i < arity; ++i) v[i] = orc_load(b[i].dtype, b[i].base, it.off[i]);
    orc_store(out->dtype, out->base, it.off[arity], run(code, n, v));
    odo_next(&it);
  }
  return E_OK;
}
