// Parity checker of the bench (NOT product code, never inside a timed region).
//
// bench.py hands the path of oracle/liboracle.so -- the plain-C restatement of
// the reference task bodies that tests/ pins against the reference itself --
// to gb_set_oracle(); the configs then recompute every verified task's output
// on the host from the same seeded inputs and compare it with what the GPU
// wrote, under SURVEY.md §8(a)'s rules:
//   exact   bit-identical (NaN payloads may differ)      add/mul/relu, i32, indexing
//   ulp1    <= 1 ulp of the output dtype                  float sums (bit-exact share reported)
//   rel     |g - w| <= tol * max(1, |w|)                  f32 softmax / f32 matmul
//   gemm32  <= 1 output ulp + k 2^-23 sum|a||b|            bf16/f16 tensor-core matmul
// The library is dlopen'ed at run time (the product never links it).
#pragma once

#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "../../oracle/gpuos_oracle.h"

namespace gbcheck {

struct Oracle {
  int (*elementwise)(int, orc_view*, orc_view*, int) = nullptr;
  int (*reduce)(int, orc_view*, orc_view*) = nullptr;
  int (*softmax)(orc_view*, orc_view*) = nullptr;
  int (*matmul)(orc_view*, orc_view*, orc_view*, int64_t) = nullptr;
  int (*program)(const orc_instr*, int, int, int, orc_view*, orc_view*, int) = nullptr;
  bool ok = false;
};

inline Oracle& oracle() {
  static Oracle o;
  return o;
}

inline bool load_oracle(const char* path) {
  Oracle& o = oracle();
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    std::fprintf(stderr, "gbcheck: cannot load %s: %s\n", path, dlerror());
    return false;
  }
  o.elementwise = reinterpret_cast<decltype(o.elementwise)>(dlsym(h, "orc_elementwise"));
  o.reduce = reinterpret_cast<decltype(o.reduce)>(dlsym(h, "orc_reduce"));
  o.softmax = reinterpret_cast<decltype(o.softmax)>(dlsym(h, "orc_softmax"));
  o.matmul = reinterpret_cast<decltype(o.matmul)>(dlsym(h, "orc_matmul"));
  o.program = reinterpret_cast<decltype(o.program)>(dlsym(h, "orc_program"));
  o.ok = o.elementwise && o.reduce && o.softmax && o.matmul && o.program;
  return o.ok;
}

inline size_t width(int dt) { return dt == ORC_F64 ? 8 : (dt == ORC_F16 || dt == ORC_BF16) ? 2 : 4; }

// A strided view of host memory for the oracle.
inline orc_view view(void* base, int dt, int64_t offset, std::initializer_list<int64_t> shape,
                     std::initializer_list<int64_t> strides) {
  orc_view v;
  std::memset(&v, 0, sizeof(v));
  v.base = base;
  v.offset = offset;
  v.dtype = v.buf_dtype = dt;
  v.rank = static_cast<int32_t>(shape.size());
  int i = 0;
  for (int64_t e : shape) v.shape[i++] = e;
  i = 0;
  for (int64_t s : strides) v.strides[i++] = s;
  return v;
}
inline orc_view view(void* base, int dt, int64_t offset, const int64_t* shape, const int64_t* strides, int rank) {
  orc_view v;
  std::memset(&v, 0, sizeof(v));
  v.base = base;
  v.offset = offset;
  v.dtype = v.buf_dtype = dt;
  v.rank = rank;
  for (int i = 0; i < rank; ++i) {
    v.shape[i] = shape[i];
    v.strides[i] = strides[i];
  }
  return v;
}

inline double decode(int dt, const void* p, int64_t i) {
  switch (dt) {
    case ORC_F32: return static_cast<const float*>(p)[i];
    case ORC_F64: return static_cast<const double*>(p)[i];
    case ORC_I32: return static_cast<const int32_t*>(p)[i];
    default: {
      const uint16_t b = static_cast<const uint16_t*>(p)[i];
      if (dt == ORC_BF16) {
        const uint32_t x = static_cast<uint32_t>(b) << 16;
        float f;
        std::memcpy(&f, &x, 4);
        return f;
      }
      // binary16
      const uint32_t e = (b >> 10) & 0x1f, m = b & 0x3ff;
      double v = e == 0 ? std::ldexp(static_cast<double>(m), -24)
                        : e == 31 ? (m ? NAN : INFINITY) : std::ldexp(static_cast<double>(m | 0x400), static_cast<int>(e) - 25);
      return (b & 0x8000) ? -v : v;
    }
  }
}
inline uint64_t bits(int dt, const void* p, int64_t i) {
  switch (width(dt)) {
    case 8: return static_cast<const uint64_t*>(p)[i];
    case 4: return static_cast<const uint32_t*>(p)[i];
    default: return static_cast<const uint16_t*>(p)[i];
  }
}
// Distance in units in the last place between two non-NaN float encodings.
inline uint64_t ulp_dist(int dt, uint64_t a, uint64_t b) {
  const int nb = static_cast<int>(width(dt)) * 8;
  const uint64_t sign = uint64_t{1} << (nb - 1);
  auto ord = [&](uint64_t x) -> int64_t {
    return (x & sign) ? -static_cast<int64_t>(x & (sign - 1)) : static_cast<int64_t>(x);
  };
  const int64_t d = ord(a) - ord(b);
  return static_cast<uint64_t>(d < 0 ? -d : d);
}
inline double out_ulp(int dt, double w) {  // spacing of the output dtype at |w|
  const double a = std::fabs(w);
  int e;
  std::frexp(a == 0 ? 1e-300 : a, &e);
  const int frac = dt == ORC_F32 ? 23 : dt == ORC_BF16 ? 7 : dt == ORC_F16 ? 10 : 52;
  const int emin = dt == ORC_F32 ? -126 : dt == ORC_BF16 ? -126 : dt == ORC_F16 ? -14 : -1022;
  return std::ldexp(1.0, std::max(e - 1, emin) - frac);
}

enum Rule { kExact, kUlp1, kRel, kGemm32 };

struct Tally {
  uint64_t tasks = 0, bad_tasks = 0, elems = 0, bad_elems = 0, bitexact = 0;
  uint64_t sum_elems = 0, sum_bitexact = 0;  // float-sum elements (the ulp1 rule)
  double max_rel = 0;
  std::string first;
  void merge(const Tally& o) {
    tasks += o.tasks;
    bad_tasks += o.bad_tasks;
    elems += o.elems;
    bad_elems += o.bad_elems;
    bitexact += o.bitexact;
    sum_elems += o.sum_elems;
    sum_bitexact += o.sum_bitexact;
    max_rel = std::max(max_rel, o.max_rel);
    if (first.empty()) first = o.first;
  }
};

// Compare n contiguous elements `got` (GPU) with `want` (oracle).  `bound`
// (kGemm32 only) holds k 2^-23 sum|a||b| per element.
inline bool compare(int dt, const void* got, const void* want, int64_t n, Rule rule, double tol, Tally& t,
                    const double* bound = nullptr, const char* what = "") {
  uint64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t gb = bits(dt, got, i), wb = bits(dt, want, i);
    const double g = decode(dt, got, i), w = decode(dt, want, i);
    const bool nan_both = std::isnan(g) && std::isnan(w);
    const bool same = gb == wb || nan_both;
    t.bitexact += same;
    if (rule == kUlp1) {
      ++t.sum_elems;
      t.sum_bitexact += same;
    }
    if (same) continue;
    bool ok = false;
    switch (rule) {
      case kExact: ok = false; break;
      case kUlp1: ok = !std::isnan(g) && !std::isnan(w) && ulp_dist(dt, gb, wb) <= 1; break;
      case kRel: {
        const double r = std::fabs(g - w) / std::max(1.0, std::fabs(w));
        t.max_rel = std::max(t.max_rel, r);
        ok = r <= tol;
        break;
      }
      case kGemm32: {
        const double lim = out_ulp(dt, w) + (bound ? bound[i] : 0.0);
        ok = std::fabs(g - w) <= lim;
        t.max_rel = std::max(t.max_rel, std::fabs(g - w) / std::max(1.0, std::fabs(w)));
        break;
      }
    }
    if (!ok) {
      if (bad == 0 && t.first.empty()) {
        char buf[256];
        std::snprintf(buf, sizeof(buf), "%s elem %lld: got %.9g want %.9g", what, static_cast<long long>(i), g, w);
        t.first = buf;
      }
      ++bad;
    }
  }
  t.elems += static_cast<uint64_t>(n);
  t.bad_elems += bad;
  ++t.tasks;
  t.bad_tasks += bad ? 1 : 0;
  return bad == 0;
}

// Run fn(i, tally) for i in [0, n) over the host's cores; returns the merged tally.
inline Tally parallel_for(size_t n, const std::function<void(size_t, Tally&)>& fn) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::atomic<size_t> next{0};
  std::vector<Tally> parts(hw);
  std::vector<std::thread> th;
  for (unsigned k = 0; k < hw; ++k)
    th.emplace_back([&, k] {
      for (;;) {
        const size_t i = next.fetch_add(64);
        if (i >= n) break;
        for (size_t j = i; j < std::min(n, i + 64); ++j) fn(j, parts[k]);
      }
    });
  for (auto& x : th) x.join();
  Tally all;
  for (const Tally& p : parts) all.merge(p);
  return all;
}

}  // namespace gbcheck
