// Tensor layer of the B200 runtime: dtypes (reference F32/F64/I32 plus F16 and
// BF16), strided views with right-aligned broadcasting, the buffer pool that
// owns device storage, host element access, and the multi-operand odometer.
// API follows reference tensor.hpp:24-325; storage and layout are new:
//   * Shape/Strides are an inline small vector, so copying a TensorView on
//     the submit path never touches the heap (rank <= 6 stays inline);
//   * BufferPool storage is CUDA managed memory obtained through the C-ABI,
//     so the pointer a task body reads is the same one BoundView writes;
//   * buffer ids index a chunked table: lookups on the submit path are
//     lock-free.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <span>
#include <sstream>
#include <string>
#include <vector>

#include "gpuos/errors.hpp"
#include "gpuos_cuda.h"

namespace gpuos {

enum class DType : uint8_t { F32 = 0, F64 = 1, I32 = 2, F16 = 3, BF16 = 4 };

inline constexpr size_t dtype_width(DType d) {
  switch (d) {
    case DType::F32: return 4;
    case DType::F64: return 8;
    case DType::I32: return 4;
    case DType::F16: return 2;
    case DType::BF16: return 2;
  }
  return 0;
}

inline const char* dtype_name(DType d) {
  switch (d) {
    case DType::F32: return "f32";
    case DType::F64: return "f64";
    case DType::I32: return "i32";
    case DType::F16: return "f16";
    case DType::BF16: return "bf16";
  }
  return "?";
}

using BufferId = uint64_t;
inline constexpr BufferId kInvalidBuffer = 0;

/// std::vector<int64_t>-like dimension list with inline storage for rank <= 6.
class Dims {
 public:
  using value_type = int64_t;
  using iterator = int64_t*;
  using const_iterator = const int64_t*;
  static constexpr uint32_t kInline = 6;

  Dims() = default;
  Dims(std::initializer_list<int64_t> il) { assign(il.begin(), il.end()); }
  Dims(size_t n, int64_t v) { assign(n, v); }
  explicit Dims(size_t n) { assign(n, 0); }
  Dims(const std::vector<int64_t>& v) { assign(v.begin(), v.end()); }  // NOLINT: implicit like the reference
  template <class It, class = decltype(*std::declval<It>())>
  Dims(It b, It e) {
    assign(b, e);
  }
  Dims(const Dims& o) { assign(o.begin(), o.end()); }
  Dims(Dims&& o) noexcept { steal(o); }
  Dims& operator=(const Dims& o) {
    if (this != &o) assign(o.begin(), o.end());
    return *this;
  }
  Dims& operator=(Dims&& o) noexcept {
    if (this != &o) {
      release();
      steal(o);
    }
    return *this;
  }
  Dims& operator=(std::initializer_list<int64_t> il) {
    assign(il.begin(), il.end());
    return *this;
  }
  ~Dims() { release(); }

  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  int64_t* data() { return heap_ ? heap_ : in_; }
  const int64_t* data() const { return heap_ ? heap_ : in_; }
  int64_t* begin() { return data(); }
  int64_t* end() { return data() + n_; }
  const int64_t* begin() const { return data(); }
  const int64_t* end() const { return data() + n_; }
  int64_t& operator[](size_t i) { return data()[i]; }
  const int64_t& operator[](size_t i) const { return data()[i]; }
  int64_t& back() { return data()[n_ - 1]; }
  const int64_t& back() const { return data()[n_ - 1]; }
  int64_t& front() { return data()[0]; }
  const int64_t& front() const { return data()[0]; }

  void reserve(size_t c) {
    if (c <= capacity()) return;
    int64_t* h = static_cast<int64_t*>(std::malloc(c * sizeof(int64_t)));
    std::memcpy(h, data(), n_ * sizeof(int64_t));
    if (heap_) std::free(heap_);
    heap_ = h;
    cap_ = static_cast<uint32_t>(c);
  }
  void push_back(int64_t v) {
    if (n_ == capacity()) reserve(capacity() * 2);
    data()[n_++] = v;
  }
  void pop_back() { --n_; }
  void clear() { n_ = 0; }
  void resize(size_t n, int64_t v = 0) {
    reserve(n);
    for (size_t i = n_; i < n; ++i) data()[i] = v;
    n_ = static_cast<uint32_t>(n);
  }
  void assign(size_t n, int64_t v) {
    n_ = 0;
    resize(n, v);
  }
  template <class It>
  void assign(It b, It e) {
    const size_t n = static_cast<size_t>(std::distance(b, e));
    n_ = 0;
    reserve(n);
    int64_t* d = data();
    for (size_t i = 0; b != e; ++b, ++i) d[i] = static_cast<int64_t>(*b);
    n_ = static_cast<uint32_t>(n);
  }
  operator std::vector<int64_t>() const { return std::vector<int64_t>(begin(), end()); }  // NOLINT
  operator std::span<const int64_t>() const { return {data(), n_}; }                     // NOLINT

  friend bool operator==(const Dims& a, const Dims& b) {
    return a.n_ == b.n_ && std::equal(a.begin(), a.end(), b.begin());
  }
  friend bool operator!=(const Dims& a, const Dims& b) { return !(a == b); }

 private:
  size_t capacity() const { return heap_ ? cap_ : kInline; }
  void release() {
    if (heap_) std::free(heap_);
    heap_ = nullptr;
    n_ = 0;
    cap_ = 0;
  }
  void steal(Dims& o) {
    n_ = o.n_;
    cap_ = o.cap_;
    heap_ = o.heap_;
    if (!heap_) std::memcpy(in_, o.in_, n_ * sizeof(int64_t));
    o.heap_ = nullptr;
    o.n_ = 0;
    o.cap_ = 0;
  }
  int64_t in_[kInline];
  int64_t* heap_ = nullptr;
  uint32_t n_ = 0;
  uint32_t cap_ = 0;
};

using Shape = Dims;
using Strides = Dims;

/// Row-major strides; the last dimension has stride 1 (reference tensor.hpp:52-62).
inline Strides contiguous_strides(std::span<const int64_t> shape) {
  Strides s(shape.size(), 0);
  int64_t acc = 1;
  for (size_t i = shape.size(); i-- > 0;) {
    s[i] = acc;
    acc *= shape[i];
  }
  return s;
}

/// Strided view of a buffer; offsets and strides in elements.
struct TensorView {
  BufferId buffer = kInvalidBuffer;
  int64_t offset = 0;
  Shape shape;
  Strides strides;
  DType dtype = DType::F32;

  size_t rank() const { return shape.size(); }
  int64_t numel() const {
    int64_t n = 1;
    for (int64_t e : shape) n *= e;
    return n;
  }
  bool is_contiguous() const {
    int64_t acc = 1;
    for (size_t i = shape.size(); i-- > 0;) {
      if (shape[i] != 1 && strides[i] != acc) return false;
      acc *= shape[i];
    }
    return true;
  }
  bool same_layout(const TensorView& o) const {
    return buffer == o.buffer && offset == o.offset && dtype == o.dtype && shape == o.shape &&
           strides == o.strides;
  }
};

inline std::string shape_to_string(std::span<const int64_t> s) {
  std::string out = "(";
  for (size_t i = 0; i < s.size(); ++i) {
    if (i) out += ",";
    out += std::to_string(s[i]);
  }
  return out + ")";
}

/// Right-aligned broadcast of two shapes (reference tensor.hpp:104-124).
inline Shape broadcast_shapes(std::span<const int64_t> a, std::span<const int64_t> b) {
  const size_t r = std::max(a.size(), b.size());
  Shape out(r, 0);
  for (size_t k = 0; k < r; ++k) {
    const int64_t x = k < a.size() ? a[a.size() - 1 - k] : 1;
    const int64_t y = k < b.size() ? b[b.size() - 1 - k] : 1;
    if (x != y && x != 1 && y != 1)
      throw Error(ErrorCode::IncompatibleShapes, shape_to_string(a) + " vs " + shape_to_string(b));
    out[r - 1 - k] = std::max(x, y);
  }
  return out;
}

/// Expand a view to `target`; broadcast dims get stride 0 (tensor.hpp:126-147).
inline TensorView broadcast_view(const TensorView& v, std::span<const int64_t> target) {
  if (v.rank() > target.size())
    throw Error(ErrorCode::IncompatibleShapes, shape_to_string(v.shape) + " to " + shape_to_string(target));
  TensorView out;
  out.buffer = v.buffer;
  out.offset = v.offset;
  out.dtype = v.dtype;
  out.shape.assign(target.begin(), target.end());
  out.strides.assign(target.size(), 0);
  const size_t rv = v.rank(), rt = target.size();
  for (size_t k = 0; k < rv; ++k) {
    const int64_t dv = v.shape[rv - 1 - k], dt = target[rt - 1 - k];
    if (dv == dt) {
      out.strides[rt - 1 - k] = v.strides[rv - 1 - k];
    } else if (dv != 1) {
      throw Error(ErrorCode::IncompatibleShapes, shape_to_string(v.shape) + " to " + shape_to_string(target));
    }
  }
  return out;
}

/// offset + sum(idx[d] * strides[d]) with bounds checks (tensor.hpp:150-165).
inline int64_t element_offset(const TensorView& v, std::span<const int64_t> idx) {
  if (idx.size() != v.rank())
    throw Error(ErrorCode::OutOfBounds,
                "index rank " + std::to_string(idx.size()) + " vs view rank " + std::to_string(v.rank()));
  int64_t off = v.offset;
  for (size_t d = 0; d < idx.size(); ++d) {
    if (idx[d] < 0 || idx[d] >= v.shape[d])
      throw Error(ErrorCode::OutOfBounds, "index " + std::to_string(idx[d]) + " out of extent " +
                                              std::to_string(v.shape[d]) + " at dim " + std::to_string(d));
    off += idx[d] * v.strides[d];
  }
  return off;
}
inline int64_t element_offset(const TensorView& v, std::initializer_list<int64_t> idx) {
  return element_offset(v, std::span<const int64_t>(idx.begin(), idx.size()));
}

// ---------------------------------------------------------------------------
// Half-precision storage conversions (round-to-nearest-even from double).
// F16/BF16 are new in this build; the narrowing rule is the reference's
// single rounding from the exact double value (tensor.hpp:354-371).
// ---------------------------------------------------------------------------
namespace detail {
inline uint16_t narrow_bits(double x, int frac_bits, int emin, int emax) {
  const uint16_t sign = std::signbit(x) ? 0x8000u : 0u;
  const int exp_shift = frac_bits;
  const int bias = emax;  // IEEE: bias == emax
  const uint16_t exp_all = static_cast<uint16_t>(((2 * bias + 1) << exp_shift));
  if (std::isnan(x)) return static_cast<uint16_t>(sign | exp_all | (1u << (frac_bits - 1)));
  const double a = std::fabs(x);
  // overflow: at or above the midpoint between the largest finite value and
  // 2^(emax+1), round-to-even goes to infinity
  const double thresh = std::ldexp(2.0 - std::ldexp(1.0, -frac_bits - 1), emax);
  if (a >= thresh) return static_cast<uint16_t>(sign | exp_all);
  if (a < std::ldexp(1.0, emin)) {
    const double q = std::nearbyint(std::ldexp(a, frac_bits - emin));
    return static_cast<uint16_t>(sign | static_cast<uint16_t>(q));
  }
  int e2 = 0;
  std::frexp(a, &e2);
  int e = e2 - 1;
  double m = std::nearbyint(std::ldexp(a, frac_bits - e));
  if (m >= std::ldexp(1.0, frac_bits + 1)) {
    m = std::ldexp(1.0, frac_bits);
    ++e;
  }
  if (e > emax) return static_cast<uint16_t>(sign | exp_all);
  const uint32_t frac = static_cast<uint32_t>(m) - (1u << frac_bits);
  return static_cast<uint16_t>(sign | ((e + bias) << exp_shift) | frac);
}
inline double widen_bits(uint16_t b, int frac_bits, int emin, int emax) {
  const bool neg = b & 0x8000u;
  const uint32_t e = (b & 0x7fffu) >> frac_bits;
  const uint32_t f = b & ((1u << frac_bits) - 1);
  const uint32_t eall = static_cast<uint32_t>(2 * emax + 1);
  double v;
  if (e == 0) {
    v = std::ldexp(static_cast<double>(f), emin - frac_bits);
  } else if (e == eall) {
    v = f ? std::nan("") : INFINITY;
  } else {
    v = std::ldexp(static_cast<double>(f | (1u << frac_bits)), static_cast<int>(e) - emax - frac_bits);
  }
  return neg ? -v : v;
}
}  // namespace detail

inline uint16_t f16_from_double(double x) { return detail::narrow_bits(x, 10, -14, 15); }
inline double f16_to_double(uint16_t b) { return detail::widen_bits(b, 10, -14, 15); }
inline uint16_t bf16_from_double(double x) { return detail::narrow_bits(x, 7, -126, 127); }
inline double bf16_to_double(uint16_t b) { return detail::widen_bits(b, 7, -126, 127); }

/// static_cast<int32_t>(double) as x86 performs it: truncation, INT32_MIN
/// out of range; the device reproduces the same rule.
inline int32_t narrow_i32(double v) {
  if (v > -2147483649.0 && v < 2147483648.0) return static_cast<int32_t>(v);
  return INT32_MIN;
}

/// What a store into `d` followed by a load yields (tensor.hpp:278-285).
inline double narrow_to(DType d, double v) {
  switch (d) {
    case DType::F32: return static_cast<double>(static_cast<float>(v));
    case DType::F64: return v;
    case DType::I32: return static_cast<double>(narrow_i32(v));
    case DType::F16: return f16_to_double(f16_from_double(v));
    case DType::BF16: return bf16_to_double(bf16_from_double(v));
  }
  return v;
}

// ---------------------------------------------------------------------------
// BufferPool: device storage through the C-ABI (or host heap when no device).
// ---------------------------------------------------------------------------
class BufferPool {
 public:
  struct Buffer {
    DType dtype = DType::F32;
    size_t length = 0;   // elements
    void* data = nullptr;
    std::atomic<bool> live{false};
  };

  BufferPool() = default;
  explicit BufferPool(gpuos_dev* dev) : dev_(dev) {}
  BufferPool(const BufferPool&) = delete;
  BufferPool& operator=(const BufferPool&) = delete;
  ~BufferPool() { clear(); }

  gpuos_dev* device() const { return dev_; }

  BufferId allocate(DType dtype, size_t length) {
    std::lock_guard<std::mutex> lk(mu_);
    void* p = nullptr;
    if (dev_) {
      uint64_t id = 0;
      check_abi(gpuos_buf_alloc(dev_, static_cast<int>(dtype), length, &id, &p), "buffer allocate");
      dev_ids_.resize(std::max<size_t>(dev_ids_.size(), next_id_ + 1), 0);
      dev_ids_[next_id_] = id;
    } else {
      const size_t bytes = std::max<size_t>(length * dtype_width(dtype), 1);
      p = std::calloc(bytes, 1);
    }
    const BufferId id = next_id_++;
    Buffer& b = slot(id, /*create=*/true);
    b.dtype = dtype;
    b.length = length;
    b.data = p;
    b.live.store(true, std::memory_order_release);
    ++count_;
    return id;
  }

  void release(BufferId id) {
    std::lock_guard<std::mutex> lk(mu_);
    Buffer* b = find(id);
    if (!b) throw Error(ErrorCode::InvalidBuffer, "release of unknown buffer " + std::to_string(id));
    b->live.store(false, std::memory_order_release);
    if (dev_) {
      gpuos_buf_free(dev_, dev_ids_[id]);
    } else {
      std::free(b->data);
    }
    b->data = nullptr;
    --count_;
  }

  /// Lock-free lookup for the submit path; nullptr when unknown/released.
  Buffer* find(BufferId id) const noexcept {
    const size_t c = static_cast<size_t>(id >> kChunkBits);
    if (id == 0 || c >= kMaxChunks) return nullptr;
    Buffer* ch = chunks_[c].load(std::memory_order_acquire);
    if (!ch) return nullptr;
    Buffer* b = &ch[id & (kChunk - 1)];
    return b->live.load(std::memory_order_acquire) ? b : nullptr;
  }

  const Buffer& lookup(BufferId id) const {
    const Buffer* b = find(id);
    if (!b) throw Error(ErrorCode::InvalidBuffer, "lookup of unknown buffer " + std::to_string(id));
    return *b;
  }
  bool contains(BufferId id) const { return find(id) != nullptr; }
  size_t length(BufferId id) const { return lookup(id).length; }
  DType dtype(BufferId id) const { return lookup(id).dtype; }
  template <typename T>
  T* data(BufferId id) {
    return static_cast<T*>(lookup(id).data);
  }
  void* raw(BufferId id) { return lookup(id).data; }
  size_t size() const { return count_.load(); }

  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t c = 0; c < kMaxChunks; ++c) {
      Buffer* ch = chunks_[c].load();
      if (!ch) continue;
      for (size_t i = 0; i < kChunk; ++i) {
        if (ch[i].live.load()) {
          ch[i].live.store(false);
          if (!dev_) std::free(ch[i].data);
          else gpuos_buf_free(dev_, dev_ids_[c * kChunk + i]);
          ch[i].data = nullptr;
        }
      }
    }
    count_ = 0;
  }

  // ---- extensions for timed runs: bulk copies and HBM residency ----
  void upload(BufferId id, const void* src, size_t bytes) {
    const Buffer& b = lookup(id);
    if (dev_) check_abi(gpuos_buf_copy(dev_, b.data, src, bytes, 0), "upload");
    else std::memcpy(b.data, src, bytes);
  }
  void download(BufferId id, void* dst, size_t bytes) const {
    const Buffer& b = lookup(id);
    if (dev_) check_abi(gpuos_buf_copy(dev_, dst, b.data, bytes, 1), "download");
    else std::memcpy(dst, b.data, bytes);
  }
  /// Bytes [byte_off, byte_off + bytes) of a buffer to the host.
  void download_range(BufferId id, size_t byte_off, void* dst, size_t bytes) const {
    const Buffer& b = lookup(id);
    if (dev_) check_abi(gpuos_buf_copy(dev_, dst, static_cast<const char*>(b.data) + byte_off, bytes, 1), "download");
    else std::memcpy(dst, static_cast<const char*>(b.data) + byte_off, bytes);
  }
  /// Byte fill of the whole buffer (benchmarks poison outputs with 0xff = NaN).
  void fill(BufferId id, int byte) {
    Buffer& b = const_cast<Buffer&>(lookup(id));
    const size_t bytes = b.length * dtype_width(b.dtype);
    if (dev_) check_abi(gpuos_buf_fill(dev_, b.data, byte, bytes), "fill");
    else std::memset(b.data, byte, bytes);
  }
  void prefetch(BufferId id) {
    if (dev_) check_abi(gpuos_buf_prefetch(dev_, dev_ids_[id]), "prefetch");
  }

 private:
  static constexpr size_t kChunkBits = 14;
  static constexpr size_t kChunk = size_t{1} << kChunkBits;
  static constexpr size_t kMaxChunks = 1u << 14;  // 268M ids

  Buffer& slot(BufferId id, bool) {
    const size_t c = static_cast<size_t>(id >> kChunkBits);
    if (c >= kMaxChunks) throw Error(ErrorCode::Internal, "buffer id space exhausted");
    Buffer* ch = chunks_[c].load(std::memory_order_acquire);
    if (!ch) {
      ch = new Buffer[kChunk];
      owned_.emplace_back(ch);
      chunks_[c].store(ch, std::memory_order_release);
    }
    return ch[id & (kChunk - 1)];
  }

  gpuos_dev* dev_ = nullptr;
  mutable std::mutex mu_;
  std::unique_ptr<std::atomic<Buffer*>[]> chunks_{new std::atomic<Buffer*>[kMaxChunks]()};
  std::vector<std::unique_ptr<Buffer[]>> owned_;
  std::vector<uint64_t> dev_ids_;  // pool id -> C-ABI buffer id
  BufferId next_id_ = 1;
  std::atomic<size_t> count_{0};
};

/// Host element access through a resolved view; loads widen to double and
/// stores narrow once (tensor.hpp:246-275).  On a device pool the storage is
/// managed memory, so this is the drop-in fill/read path of the reference
/// tests; timed runs use BufferPool::upload/download instead.
struct BoundView {
  void* base = nullptr;
  const TensorView* view = nullptr;

  BoundView() = default;
  BoundView(BufferPool& pool, const TensorView& v) : view(&v) {
    const auto& buf = pool.lookup(v.buffer);
    if (buf.dtype != v.dtype) throw Error(ErrorCode::DTypeMismatch, "view dtype does not match buffer dtype");
    base = buf.data;
  }

  double load(int64_t elem) const {
    switch (view->dtype) {
      case DType::F32: return static_cast<double>(static_cast<const float*>(base)[elem]);
      case DType::F64: return static_cast<const double*>(base)[elem];
      case DType::I32: return static_cast<double>(static_cast<const int32_t*>(base)[elem]);
      case DType::F16: return f16_to_double(static_cast<const uint16_t*>(base)[elem]);
      case DType::BF16: return bf16_to_double(static_cast<const uint16_t*>(base)[elem]);
    }
    return 0.0;
  }
  void store(int64_t elem, double value) const {
    switch (view->dtype) {
      case DType::F32: static_cast<float*>(base)[elem] = static_cast<float>(value); break;
      case DType::F64: static_cast<double*>(base)[elem] = value; break;
      case DType::I32: static_cast<int32_t*>(base)[elem] = narrow_i32(value); break;
      case DType::F16: static_cast<uint16_t*>(base)[elem] = f16_from_double(value); break;
      case DType::BF16: static_cast<uint16_t*>(base)[elem] = bf16_from_double(value); break;
    }
  }
};

/// Row-major odometer over a shape tracking one element offset per operand
/// (tensor.hpp:289-325).
class IndexIterator {
 public:
  IndexIterator(std::span<const int64_t> shape, std::span<const TensorView* const> operands)
      : shape_(shape.begin(), shape.end()), idx_(shape.size(), 0) {
    for (const TensorView* v : operands) {
      offsets_.push_back(v->offset);
      strides_.push_back(v->strides);
    }
    count_ = 1;
    for (int64_t e : shape_) count_ *= e;
  }
  int64_t count() const { return count_; }
  int64_t offset(size_t operand) const { return offsets_[operand]; }
  std::span<const int64_t> index() const { return idx_; }
  bool next() {
    for (size_t d = shape_.size(); d-- > 0;) {
      ++idx_[d];
      for (size_t o = 0; o < offsets_.size(); ++o) offsets_[o] += strides_[o][d];
      if (idx_[d] < shape_[d]) return true;
      for (size_t o = 0; o < offsets_.size(); ++o) offsets_[o] -= strides_[o][d] * shape_[d];
      idx_[d] = 0;
    }
    return false;
  }

 private:
  Shape shape_;
  Shape idx_;
  std::vector<int64_t> offsets_;
  std::vector<Strides> strides_;
  int64_t count_ = 1;
};

}  // namespace gpuos
