// gpuos::Runtime — the drop-in host API (reference runtime.hpp:205-450) over
// the B200 C-ABI.  One producer thread submits; handles may be waited on from
// any thread (reference threading contract, runtime.hpp:5-9).
//
// Submission path (the north-star hot path, producer side):
//   validate -> eligible -> reserve a ring slot -> resolve views to device
//   addresses -> publish the 384-byte descriptor (streaming stores + release)
//   The persistent worker kernel claims, dispatches through the dual-bank
//   device table and posts the task's completion word, which the TaskHandle
//   reads directly: no completion thread, no handle map, no allocation for
//   rank <= 6 views.
// Ineligible calls and queue-full overflow take the conventional path: one
// cudaLaunchKernel of the same task body, synchronous (runtime.hpp:567-619).
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <span>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

#include <immintrin.h>

#include "gpuos/bytecode.hpp"
#include "gpuos/errors.hpp"
#include "gpuos_ring_format.h"
#include "gpuos/expr.hpp"
#include "gpuos/opcompiler.hpp"
#include "gpuos/ops.hpp"
#include "gpuos/optable.hpp"
#include "gpuos/queue.hpp"
#include "gpuos/telemetry.hpp"
#include "gpuos/tensor.hpp"
#include "gpuos_cuda.h"

namespace gpuos {

inline constexpr uint32_t kCompositeOpId = GPUOS_COMPOSITE_OP_ID;

enum class TaskState : uint8_t { Pending = 0, Done = 1, Failed = 2 };

inline const char* task_state_name(TaskState s) {
  switch (s) {
    case TaskState::Pending: return "Pending";
    case TaskState::Done: return "Done";
    case TaskState::Failed: return "Failed";
  }
  return "unknown";
}

inline uint64_t monotonic_ns() {
  return static_cast<uint64_t>(
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
          .count());
}

namespace detail {

/// Dataflow key of an expression (runtime.hpp:92-126's role): fused chains
/// with different dataflow never share a compiled program.  Prefix form;
/// constants print with 17 significant digits, so distinct values differ.
inline void canonical_expr(const Expr& e, std::string& out) {
  char buf[48];
  switch (e.kind) {
    case ExprKind::Const:
      std::snprintf(buf, sizeof(buf), "c%.17g", e.value);
      out += buf;
      return;
    case ExprKind::In:
      out += "i" + std::to_string(e.index);
      return;
    case ExprKind::Param:
      out += "p" + std::to_string(e.index);
      return;
    case ExprKind::Narrow:
      out += "nw" + std::to_string(static_cast<int>(e.narrow_dtype));
      break;
    default:
      out += std::to_string(static_cast<int>(e.kind));
  }
  out += '(';
  if (e.a) canonical_expr(*e.a, out);
  if (e.b) {
    out += ',';
    canonical_expr(*e.b, out);
  }
  out += ')';
}

/// Completion cells: 8-byte words in mapped pinned memory, one per live task,
/// written exactly once (device st.release.sys, or the host on the inline and
/// validation paths).  Replaces HandleState (runtime.hpp:59-88).  Reference
/// counts are host-only; a cell is reusable once unreferenced and completed.
class CellPool {
 public:
  static constexpr uint32_t kBlockBits = 16;
  static constexpr uint32_t kBlock = 1u << kBlockBits;
  /// Blocks live at fixed addresses for the pool's lifetime: the producer
  /// appends (grow) while any thread may wait on a handle, so readers index a
  /// fixed array of atomically published Block pointers, never a container
  /// that could reallocate under them.  256 blocks = 16M live cells.
  static constexpr uint32_t kMaxBlocks = 256;

  explicit CellPool(gpuos_dev* dev) : dev_(dev) { grow(); }

  uint64_t* word(uint32_t g) const {
    return blk(g)->host.load(std::memory_order_acquire) + (g & (kBlock - 1));
  }

  /// Completion record of cell g for fused composites (mapped pinned, 32
  /// words: n, then (cell device address, seq) pairs); allocated per block
  /// on first use.  Only the composite's final cell owns one; the device reads
  /// the record before it posts that final cell, and a cell (with its record)
  /// is not reused before its task completes, so records never race.
  static constexpr uint32_t kRecordWords = 32;
  uint64_t* record(uint32_t g, uint64_t* device_addr) {
    Block& b = *blk(g);
    if (!b.rec_host) check_abi(gpuos_cells_alloc(dev_, kBlock * kRecordWords, &b.rec_host, &b.rec_dev), "records");
    const uint64_t i = g & (kBlock - 1);
    *device_addr = b.rec_dev + 8ull * kRecordWords * i;
    return b.rec_host + kRecordWords * i;
  }
  uint64_t device_addr(uint32_t g) const { return blk(g)->dev + 8ull * (g & (kBlock - 1)); }

  /// Producer thread only.  A cell is reusable when no handle references it
  /// and its previous task's completion (tagged with that task's seq) has
  /// landed; words are seq-tagged, so a reused cell needs no clearing store.
  uint32_t acquire(uint64_t seq) {
    const uint32_t total = nblocks_.load(std::memory_order_relaxed) * kBlock;
    for (int probe = 0; probe < 64; ++probe) {
      const uint32_t g = cursor_;
      cursor_ = (cursor_ + 1) % total;
      {  // the device wrote these words over PCIe: fetch them ahead of use
        const uint32_t ahead = (g + 32) % total;
        _mm_prefetch(reinterpret_cast<const char*>(word(ahead)), _MM_HINT_T0);
      }
      Block& b = *blk(g);
      const uint32_t i = g & (kBlock - 1);
      if (b.refs[i].load(std::memory_order_acquire) != 0) continue;
      const uint64_t prev = b.last_seq[i];
      if (prev != 0) {
        const uint64_t w = __atomic_load_n(&b.host.load(std::memory_order_relaxed)[i], __ATOMIC_ACQUIRE);
        if ((w & 0xffu) == 0 || (w >> 16) != (prev & kSeqMask)) continue;  // previous task in flight
      }
      b.last_seq[i] = seq;
      // the caller's handle adopts this first reference: a plain store, since
      // no handle can name a cell whose count is zero (one RMW saved per task)
      b.refs[i].store(1, std::memory_order_relaxed);
      return g;
    }
    cursor_ = nblocks_.load(std::memory_order_relaxed) * kBlock;
    grow();
    const uint32_t g = cursor_;
    cursor_ = (cursor_ + 1) % (nblocks_.load(std::memory_order_relaxed) * kBlock);
    blk(g)->last_seq[g & (kBlock - 1)] = seq;
    blk(g)->refs[g & (kBlock - 1)].store(1, std::memory_order_relaxed);
    return g;
  }
  static constexpr uint64_t kSeqMask = (uint64_t{1} << 48) - 1;
  // One atomic per handle copy/destroy: the pool's own lifetime after the
  // runtime is gone is derived from the per-cell counts (try_delete), not
  // from a second shared counter.
  void addref(uint32_t g) { blk(g)->refs[g & (kBlock - 1)].fetch_add(1, std::memory_order_relaxed); }
  void release(uint32_t g) {
    // seq_cst pairs with orphan(): the last releaser or orphan() sees the other
    if (blk(g)->refs[g & (kBlock - 1)].fetch_sub(1, std::memory_order_seq_cst) == 1 &&
        orphaned_.load(std::memory_order_seq_cst))
      try_delete();
  }
  long use_count(uint32_t g) const {
    return static_cast<long>(blk(g)->refs[g & (kBlock - 1)].load(std::memory_order_relaxed));
  }
  /// Host-side completion (inline / validation / shutdown paths).
  void complete(uint32_t g, uint64_t seq, ErrorCode c) {
    const uint64_t w = (c == ErrorCode::Ok ? 1u : 2u) | (static_cast<uint64_t>(c) << 8) | (seq << 16);
    __atomic_store_n(word(g), w, __ATOMIC_RELEASE);
  }
  /// Before the device memory goes away: copy words to the heap, then free
  /// ourselves when the last handle drops.  Readers switch to the heap copy
  /// through the atomic host pointer.
  void orphan() {
    const uint32_t n = nblocks_.load(std::memory_order_acquire);
    for (uint32_t k = 0; k < n; ++k) {
      Block& b = *blocks_[k].load(std::memory_order_acquire);
      uint64_t* h = new uint64_t[kBlock];
      std::memcpy(h, b.host.load(std::memory_order_relaxed), kBlock * 8);
      b.heap = h;
      b.host.store(h, std::memory_order_release);
    }
    orphaned_.store(true, std::memory_order_seq_cst);
    try_delete();
  }
  ~CellPool() {
    const uint32_t n = nblocks_.load(std::memory_order_acquire);
    for (uint32_t k = 0; k < n; ++k) {
      Block* b = blocks_[k].load(std::memory_order_acquire);
      delete[] b->heap;
      delete[] b->refs;
      delete[] b->last_seq;
      delete b;
    }
  }
  uint32_t blocks() const { return nblocks_.load(std::memory_order_acquire); }
  /// Intentional no-consumer windows (generation handovers, shutdown) nest.
  void pause(int delta) { paused_.fetch_add(delta, std::memory_order_acq_rel); }
  /// True when no worker generation is resident outside an intentional
  /// window: a waiter on a pending cell would otherwise spin forever.
  bool consumer_lost() const {
    if (orphaned_.load(std::memory_order_acquire) || paused_.load(std::memory_order_acquire) > 0) return false;
    return gpuos_dev_alive(dev_) == 0 && paused_.load(std::memory_order_acquire) == 0;
  }

 private:
  struct Block {
    std::atomic<uint64_t*> host{nullptr};
    uint64_t dev = 0;
    std::atomic<uint32_t>* refs = nullptr;
    uint64_t* last_seq = nullptr;  // seq of the cell's latest task, 0 = never used
    uint64_t* rec_host = nullptr;  // fused-composite completion records (lazily)
    uint64_t rec_dev = 0;
    uint64_t* heap = nullptr;      // orphaned copy of the words
  };
  Block* blk(uint32_t g) const { return blocks_[g >> kBlockBits].load(std::memory_order_acquire); }
  void grow() {
    const uint32_t n = nblocks_.load(std::memory_order_relaxed);
    if (n >= kMaxBlocks) throw Error(ErrorCode::Internal, "completion cells exhausted (16M live handles)");
    Block* b = new Block;
    uint64_t* host = nullptr;
    check_abi(gpuos_cells_alloc(dev_, kBlock, &host, &b->dev), "cells");
    b->host.store(host, std::memory_order_relaxed);
    b->refs = new std::atomic<uint32_t>[kBlock]();
    b->last_seq = new uint64_t[kBlock]();
    blocks_[n].store(b, std::memory_order_release);  // published before any cell of it is handed out
    nblocks_.store(n + 1, std::memory_order_release);
  }

  // After orphan(): delete once no handle references any cell.
  void try_delete() {
    const uint32_t n = nblocks_.load(std::memory_order_acquire);
    for (uint32_t k = 0; k < n; ++k) {
      const Block& b = *blocks_[k].load(std::memory_order_acquire);
      for (uint32_t i = 0; i < kBlock; ++i)
        if (b.refs[i].load(std::memory_order_seq_cst) != 0) return;
    }
    if (!deleting_.exchange(true, std::memory_order_acq_rel)) delete this;
  }

  gpuos_dev* dev_;
  std::array<std::atomic<Block*>, kMaxBlocks> blocks_{};
  std::atomic<uint32_t> nblocks_{0};
  uint32_t cursor_ = 0;
  std::atomic<bool> orphaned_{false};
  std::atomic<bool> deleting_{false};
  std::atomic<int> paused_{0};
};

}  // namespace detail

/// Completion token (runtime.hpp:130-162).  Reads the task's completion word.
class TaskHandle {
 public:
  TaskHandle() = default;
  TaskHandle(const TaskHandle& o) : pool_(o.pool_), cell_(o.cell_), id_(o.id_) { ref(); }
  TaskHandle(TaskHandle&& o) noexcept : pool_(o.pool_), cell_(o.cell_), id_(o.id_) { o.pool_ = nullptr; }
  TaskHandle& operator=(const TaskHandle& o) {
    if (this != &o) {
      unref();
      pool_ = o.pool_;
      cell_ = o.cell_;
      id_ = o.id_;
      ref();
    }
    return *this;
  }
  TaskHandle& operator=(TaskHandle&& o) noexcept {
    if (this != &o) {
      unref();
      pool_ = o.pool_;
      cell_ = o.cell_;
      id_ = o.id_;
      o.pool_ = nullptr;
    }
    return *this;
  }
  ~TaskHandle() { unref(); }

  bool valid() const { return pool_ != nullptr; }
  uint64_t id() const {
    check();
    return id_;
  }
  TaskState state() const { return static_cast<TaskState>(raw() & 0xffu); }
  /// Ok while Pending or Done; the failure code once Failed.
  ErrorCode error() const {
    const uint64_t w = raw();
    if ((w & 0xffu) != static_cast<uint64_t>(TaskState::Failed)) return ErrorCode::Ok;
    return static_cast<ErrorCode>((w >> 8) & 0xffu);
  }
  /// Block until terminal: spin, then yield, then sleep.  Throws
  /// RuntimeStopped when the worker generation is gone (twice, ~10 ms apart)
  /// while the task is still pending, instead of spinning forever.
  TaskState wait() const {
    uint64_t w = raw();
    int lost = 0;
    for (uint32_t spin = 0; (w & 0xffu) == 0; ++spin) {
      if (spin < 2048) {
        __builtin_ia32_pause();
      } else if (spin < 4096) {
        std::this_thread::yield();
      } else {
        std::this_thread::sleep_for(std::chrono::microseconds(10));
        if ((spin & 1023) == 0) {
          lost = pool_->consumer_lost() ? lost + 1 : 0;
          if (lost >= 2 && (raw() & 0xffu) == 0)
            throw Error(ErrorCode::RuntimeStopped, "worker generation stopped with the task pending");
        }
      }
      w = raw();
    }
    return static_cast<TaskState>(w & 0xffu);
  }
  long use_count() const { return pool_ ? pool_->use_count(cell_) : 0; }

 private:
  friend class Runtime;
  // adopts the reference CellPool::acquire stored for it
  TaskHandle(detail::CellPool* p, uint32_t cell, uint64_t id) : pool_(p), cell_(cell), id_(id) {}
  void check() const {
    if (!pool_) throw Error(ErrorCode::Internal, "operation on an invalid task handle");
  }
  // The cell word belongs to this task only when its seq tag matches.
  uint64_t raw() const {
    check();
    const uint64_t w = __atomic_load_n(pool_->word(cell_), __ATOMIC_ACQUIRE);
    return (w >> 16) == (id_ & detail::CellPool::kSeqMask) ? w : 0;
  }
  void ref() {
    if (pool_) pool_->addref(cell_);
  }
  void unref() {
    if (pool_) pool_->release(cell_);
    pool_ = nullptr;
  }
  detail::CellPool* pool_ = nullptr;
  uint32_t cell_ = 0;
  uint64_t id_ = 0;
};

struct OpCall {
  uint64_t op_id = 0;
  std::vector<TensorView> inputs;
  TensorView output;
  std::vector<double> scalars;
};

struct WorkerConfig {
  size_t num_workers = 0;         // worker CTAs; 0 = one per SM
  uint64_t yield_every = 0;       // executor.hpp:28
  uint32_t spin_iterations = 64;  // executor.hpp:29
  uint32_t backoff_max_exp = 6;   // nanosleep ladder 64 ns * 2^k
};

struct RuntimeConfig {
  size_t capacity = 4096;
  WorkerConfig workers;
  uint64_t max_elements = 65536;
  int64_t max_sdpa_context = 2048;
  bool fusion_enabled = false;
  size_t max_chain = 8;
  size_t table_slots = 1024;
  size_t trace_capacity = 65536;
  bool telemetry_enabled = true;
  int device = 0;
  /// Route matmul_small / vecmat (dims <= 256) to the persistent workers.  The
  /// reference never queues them (runtime.hpp:531-534); config 3 needs them
  /// queued, so this build defaults to true.
  bool queue_matmul = true;
  /// Task buffers in plain device memory instead of managed memory (faster
  /// host<->device copies; host access only through pool().upload/download).
  bool device_buffers = false;
  /// Backpressure before the queue-full fallback: how long submit keeps
  /// retrying a full ring before it runs the task inline (runtime.hpp:562-564
  /// falls back at once).  The inline path here is a kernel launch + sync
  /// (~15 us), while the workers free a slot every few hundred ns, so a short
  /// wait is the cheaper way to absorb a producer that outruns the device.
  /// 0 = the reference's immediate fallback.  Env GPUOS_QUEUE_SPIN_NS.
  uint64_t queue_full_spin_ns = 50000;

  /// GPUOS_CAPACITY, GPUOS_WORKERS, GPUOS_YIELD_EVERY, GPUOS_MAX_ELEMS, GPUOS_DEVICE.
  static RuntimeConfig from_env() {
    RuntimeConfig c;
    c.capacity = static_cast<size_t>(env_u64("GPUOS_CAPACITY", c.capacity));
    c.workers.num_workers = static_cast<size_t>(env_u64("GPUOS_WORKERS", c.workers.num_workers));
    c.workers.yield_every = env_u64("GPUOS_YIELD_EVERY", c.workers.yield_every);
    c.max_elements = env_u64("GPUOS_MAX_ELEMS", c.max_elements);
    c.device = static_cast<int>(env_u64("GPUOS_DEVICE", static_cast<uint64_t>(c.device)));
    c.queue_full_spin_ns = env_u64("GPUOS_QUEUE_SPIN_NS", c.queue_full_spin_ns);
    return c;
  }

 private:
  static uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* s = std::getenv(name);
    if (!s || !*s) return dflt;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(s, &end, 10);
    return (end == s || *end != '\0') ? dflt : static_cast<uint64_t>(v);
  }
};

class Runtime {
 public:
  explicit Runtime(RuntimeConfig cfg = {}) : cfg_(normalize(std::move(cfg))) {
    if (cfg_.capacity == 0) throw Error(ErrorCode::ZeroCapacity, "queue capacity must be positive");
    gpuos_cfg c{};
    gpuos_default_cfg(&c);
    c.capacity = cfg_.capacity;
    c.table_slots = static_cast<uint32_t>(cfg_.table_slots);
    c.num_workers = static_cast<uint32_t>(cfg_.workers.num_workers);
    c.spin_iterations = cfg_.workers.spin_iterations;
    c.backoff_max_exp = cfg_.workers.backoff_max_exp;
    c.yield_every = cfg_.workers.yield_every;
    c.trace_capacity = cfg_.trace_capacity;
    c.telemetry = cfg_.telemetry_enabled ? 1u : 0u;
    c.flags = cfg_.device_buffers ? GPUOS_CFG_DEVICE_BUFFERS : 0u;
    check_abi(gpuos_dev_open(cfg_.device, &c, &dev_), "gpuos_dev_open");
    check_abi(gpuos_ring_view_get(dev_, &ring_), "gpuos_ring_view_get");
    pool_ = std::make_unique<BufferPool>(dev_);
    table_ = std::make_unique<OperatorTable>(dev_);
    cells_ = new detail::CellPool(dev_);
    counters_ = std::make_unique<Counters>(cfg_.table_slots < 256 ? cfg_.table_slots : 256);
    check_abi(gpuos_stream_create(dev_, &inline_stream_), "inline stream");
    // builtins at their fixed ids, then the composite handler: version 15
    // after construction, as in the reference (test_runtime.cpp:61-62).
    for (uint32_t i = 0; i < kNumBuiltinOps; ++i) {
      InjectionRecord meta;
      meta.template_name = "builtin";
      meta.signature = op_kind_name(static_cast<OpKind>(i));
      table_->install_builtin(i, static_cast<OpKind>(i), std::move(meta));
    }
    InjectionRecord cm;
    cm.template_name = "builtin";
    cm.signature = "composite";
    table_->install_program(kCompositeOpId, composite_placeholder(), 1, DType::F64, std::move(cm));
    fusion_on_ = cfg_.fusion_enabled;
  }

  ~Runtime() {
    shutdown();
    if (inline_stream_) gpuos_stream_destroy(dev_, inline_stream_);
    table_.reset();
    pool_.reset();
    cells_->orphan();
    gpuos_dev_close(dev_);
  }

  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;

  // ---- tensors ----
  BufferPool& pool() { return *pool_; }
  TensorView alloc_tensor(DType dtype, Shape shape) {
    TensorView v;
    v.dtype = dtype;
    v.shape = std::move(shape);
    v.strides = contiguous_strides(v.shape);
    v.buffer = pool_->allocate(dtype, static_cast<size_t>(v.numel()));
    return v;
  }

  // ---- submission (never throws; failures land on the handle) ----
  TaskHandle submit(uint64_t op_id, std::vector<TensorView> inputs, TensorView output,
                    std::vector<double> scalars = {}) {
    return submit_span(op_id, inputs, output, scalars);
  }
  TaskHandle submit(OpKind kind, std::vector<TensorView> inputs, TensorView output, std::vector<double> scalars = {}) {
    return submit_span(static_cast<uint64_t>(kind), inputs, output, scalars);
  }
  /// Braced-list fast path: `rt.submit(OpKind::Add, {a, b}, c)` allocates nothing.
  TaskHandle submit(OpKind kind, std::initializer_list<TensorView> inputs, const TensorView& output,
                    std::initializer_list<double> scalars = {}) {
    return submit_span(static_cast<uint64_t>(kind), std::span<const TensorView>(inputs.begin(), inputs.size()), output,
                       std::span<const double>(scalars.begin(), scalars.size()));
  }
  TaskHandle submit(uint64_t op_id, std::initializer_list<TensorView> inputs, const TensorView& output,
                    std::initializer_list<double> scalars = {}) {
    return submit_span(op_id, std::span<const TensorView>(inputs.begin(), inputs.size()), output,
                       std::span<const double>(scalars.begin(), scalars.size()));
  }
  TaskHandle submit(const OpCall& call) { return submit_span(call.op_id, call.inputs, call.output, call.scalars); }

  TaskHandle submit_span(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
                         std::span<const double> scalars) {
    const uint64_t id = next_id_++;
    const uint32_t cell = cells_->acquire(id);
    TaskHandle h(cells_, cell, id);
    if (stopped_) {
      counters_->inc_failed();
      cells_->complete(cell, id, ErrorCode::RuntimeStopped);
      return h;
    }
    if (const ErrorCode v = validate(inputs, output, scalars); v != ErrorCode::Ok) {
      counters_->inc_failed();  // not counted as submitted (runtime.hpp:261-265)
      cells_->complete(cell, id, v);
      return h;
    }
    counters_->inc_submitted();
    const bool elig = eligible(op_id, inputs, output);
    // fusion (runtime.hpp:270-281): chainable elementwise steps accumulate
    if (fusion_on_ && elig && scalars.empty() && chainable(op_id, inputs, output)) {
      if (chain_try_append(op_id, inputs, output, cell, id)) {
        if (chain_.size() >= std::min<size_t>(cfg_.max_chain, GPUOS_MAX_FUSED + 1)) flush_chain();
        return h;
      }
      flush_chain();
      if (chain_try_append(op_id, inputs, output, cell, id)) {
        if (chain_.size() >= std::min<size_t>(cfg_.max_chain, GPUOS_MAX_FUSED + 1)) flush_chain();
        return h;
      }
    }
    if (!chain_.empty()) flush_chain();  // later work must observe chained writes
    route(op_id, inputs, output, scalars, cell, id, elig, 0);
    return h;
  }

  // ---- fusion (runtime.hpp:296-327, 641-933) ----
  /// Accumulate elementwise chains on submit; turning fusion off flushes.
  void set_fusion(bool on) {
    if (!on) flush_chain();
    fusion_on_ = on;
  }
  bool fusion() const { return fusion_on_; }
  /// Flush the pending chain; a no-op when nothing is chained.
  void fuse() { flush_chain(); }
  /// Submit a whole chain and flush it as one unit (intermediates elided
  /// unless a handle other than the returned one is retained).
  std::vector<TaskHandle> fuse(std::span<const OpCall> calls) {
    const bool prev_on = fusion_on_;
    const long prev_base = chain_handle_baseline_;
    fusion_on_ = true;
    chain_handle_baseline_ = 1;  // the returned vector holds one reference
    std::vector<TaskHandle> out;
    out.reserve(calls.size());
    for (const OpCall& c : calls) out.push_back(submit(c));
    flush_chain();
    chain_handle_baseline_ = prev_base;
    fusion_on_ = prev_on;
    return out;
  }
  /// Submissions folded into composites; submitted == inline + committed + absorbed.
  uint64_t fusion_absorbed() const { return fusion_absorbed_; }

  // ---- injection ----
  uint64_t inject_operator(const std::string& template_name, std::span<const double> params = {},
                           DType dtype = DType::F32) {
    if (next_injected_id_ >= table_->slots()) throw Error(ErrorCode::TableFull, "no free injected op ids");
    return inject_operator_at(static_cast<uint32_t>(next_injected_id_), template_name, params, dtype);
  }
  uint64_t inject_operator_at(uint32_t op_id, const std::string& template_name, std::span<const double> params = {},
                              DType dtype = DType::F32) {
    NvtxRange nvtx_("gpuos::inject_operator_at");
    if (stopped_) throw Error(ErrorCode::RuntimeStopped, "inject after shutdown");
    if (op_id < kFirstInjectedId)
      throw Error(ErrorCode::OutOfRange, "injected ids start at " + std::to_string(kFirstInjectedId));
    if (op_id >= table_->slots())
      throw Error(ErrorCode::OutOfRange, "op id " + std::to_string(op_id) + " past table size");
    const OperatorTemplate tmpl = registry_.get(template_name);
    const uint64_t h0 = cache_.hits(), m0 = cache_.misses();
    ModulePtr mod;
    try {
      mod = cache_.compile_or_get(tmpl, params, dtype);
    } catch (...) {
      sync_cache_counters(h0, m0);
      throw;
    }
    sync_cache_counters(h0, m0);
    InjectionRecord meta;
    meta.template_name = template_name;
    meta.params.assign(params.begin(), params.end());
    meta.signature = signature_key(mod->signature);
    last_inject_ = table_->install_program(op_id, mod->bytecode, mod->signature.arity, dtype, std::move(meta));
    modules_by_id_[op_id] = mod;
    counters_->inc_injections();
    if (op_id >= next_injected_id_) next_injected_id_ = static_cast<uint64_t>(op_id) + 1;
    return op_id;
  }
  void kill_operator(uint32_t op_id) {
    NvtxRange nvtx_("gpuos::kill_operator");
    if (stopped_) throw Error(ErrorCode::RuntimeStopped, "kill after shutdown");
    table_->kill(op_id);
    modules_by_id_.erase(op_id);  // killed injected ops leave the eligible set
  }
  /// Timings of the most recent injection's upload / epoch wait / bank write / flip.
  const gpuos_inject_stats& last_inject_stats() const { return last_inject_; }

  /// Phases of the most recent native promotion (ns).
  struct NativeStats {
    uint64_t codegen_ns = 0, compile_ns = 0, link_ns = 0;
    gpuos_native_stats handover{};  // drain / module load / relaunch
    gpuos_inject_stats install{};   // table flip
    bool compiled = false;          // false: the object came from the native cache
  };
  const NativeStats& last_native_stats() const { return last_native_; }

  /// Promote injected operator `op_id` from its device program to native
  /// code: CUDA C++ generated from the verified program (same fp64 operations
  /// in the same order, one rounding on store), NVRTC -> relocatable sm_100a
  /// object (cached per signature), nvJitLink with the relocatable worker
  /// image and every other promoted op, module load at a generation handover,
  /// then a dual-bank flip of the entry to the native kind.  Throws
  /// gpuos::Error on compile/link/load failures; the op keeps running its
  /// program until the flip.
  void promote_native(uint32_t op_id) {
    NvtxRange nvtx_("gpuos::promote_native");
    if (stopped_) throw Error(ErrorCode::RuntimeStopped, "promote after shutdown");
    auto it = modules_by_id_.find(op_id);
    if (it == modules_by_id_.end()) throw Error(ErrorCode::NotInstalled, "op " + std::to_string(op_id) + " is not injected");
    const ModulePtr mod = it->second;
    NativeStats st;
    uint32_t slot;
    if (auto sl = native_slot_.find(op_id); sl != native_slot_.end()) {
      slot = sl->second;
    } else {
      if (native_slot_.size() >= GPUOS_NATIVE_SLOTS) throw Error(ErrorCode::TableFull, "no free native slots");
      slot = static_cast<uint32_t>(native_slot_.size());
      native_slot_[op_id] = slot;
    }
    const std::string key = signature_key(mod->signature);
    auto obj = native_cache_.find(key);
    if (obj == native_cache_.end()) {
      const uint64_t t0 = monotonic_ns();
      const std::string src = native_source(mod->bytecode, mod->signature.arity, mod->signature.dtype, key);
      const uint64_t t1 = monotonic_ns();
      void* o = nullptr;
      size_t n = 0;
      uint64_t cns = 0;
      std::string log(16384, '\0');
      const int rc = gpuos_jit_compile_object(src.c_str(), &o, &n, &cns, log.data(), log.size());
      if (rc != 0) throw Error(static_cast<ErrorCode>(rc), "native compile failed: " + std::string(log.c_str()));
      obj = native_cache_.emplace(key, std::string(static_cast<const char*>(o), n)).first;
      gpuos_free(o);
      st.codegen_ns = t1 - t0;
      st.compile_ns = cns;
      st.compiled = true;
    }
    native_obj_[slot] = key;
    // link the worker image with every promoted op's object
    std::vector<const void*> objs;
    std::vector<size_t> sizes;
    std::vector<uint32_t> slots;
    std::vector<std::string> syms;
    for (const auto& [s_, k_] : native_obj_) {
      const std::string& bytes = native_cache_.at(k_);
      objs.push_back(bytes.data());
      sizes.push_back(bytes.size());
      slots.push_back(s_);
      syms.push_back(native_symbol(k_));
    }
    void* cubin = nullptr;
    size_t csize = 0;
    std::string log(16384, '\0');
    int rc = gpuos_jit_link_worker(objs.data(), sizes.data(), static_cast<int>(objs.size()), &cubin, &csize,
                                   &st.link_ns, log.data(), log.size());
    if (rc != 0) throw Error(static_cast<ErrorCode>(rc), "native link failed: " + std::string(log.c_str()));
    std::vector<const char*> sym_ptrs;
    for (const std::string& x : syms) sym_ptrs.push_back(x.c_str());
    cells_->pause(1);  // the handover's drain/relaunch window
    rc = gpuos_dev_load_native(dev_, cubin, csize, slots.data(), sym_ptrs.data(), static_cast<int>(slots.size()),
                               &st.handover);
    cells_->pause(-1);
    gpuos_free(cubin);
    if (rc != 0) throw Error(static_cast<ErrorCode>(rc), "native module load failed");
    InjectionRecord meta;
    meta.template_name = mod->signature.template_name;
    meta.params.assign(mod->signature.params.begin(), mod->signature.params.end());
    meta.signature = key + " [native]";
    st.install = table_->install_native(op_id, slot, mod->bytecode, mod->signature.arity, mod->signature.dtype,
                                        std::move(meta));
    last_native_ = st;
  }
  bool is_native(uint32_t op_id) const { return native_slot_.count(op_id) != 0; }

  TemplateRegistry& templates() { return registry_; }
  OperatorTable& table() { return *table_; }
  ModuleCache& module_cache() { return cache_; }

  // ---- completion / introspection ----
  TaskState wait(const TaskHandle& h) {
    if (!chain_.empty()) flush_chain();  // runtime.hpp:392-395
    return h.wait();
  }
  /// Device-side ordering (extension: the reference orders tasks only through
  /// host waits, runtime.hpp:7-9).  Every task submitted after fence() starts
  /// only after every task submitted before it has completed; the producer
  /// does not block -- the worker that claims a later task waits on the
  /// device's processed count.  Lasts until the next fence() or wait_all().
  void fence() {
    NvtxRange nvtx_("gpuos::fence");
    if (!chain_.empty()) flush_chain();
    fence_target_ = committed_tasks_;
    fence_on_ = true;
  }
  void wait_all() {
    NvtxRange nvtx_("gpuos::wait_all");
    if (!chain_.empty()) flush_chain();
    const int rc = gpuos_ring_wait_processed(dev_, committed_tasks_);
    if (rc == 0) fence_on_ = false;  // everything before any fence is done
    if (rc == static_cast<int>(ErrorCode::RuntimeStopped) && !stopped_)
      throw Error(ErrorCode::RuntimeStopped, "worker generation stopped with tasks pending");
    if (rc != 0 && rc != static_cast<int>(ErrorCode::RuntimeStopped)) check_abi(rc, "wait_all");
  }
  TaskQueue::Snapshot peek_queue() const {
    gpuos_snapshot s{};
    gpuos_ring_peek(dev_, &s);
    return TaskQueue::Snapshot{s.head, s.tail, s.processed};
  }
  CounterSnapshot counters() const {
    CounterSnapshot s = counters_->snapshot();
    gpuos_dev_stats d{};
    if (gpuos_dev_get_stats(dev_, &d) == 0) {
      s.processed = d.processed;
      s.stalls = d.stalls;
      s.failed += d.failed;
      for (size_t i = 0; i < 256; ++i) {
        if (!d.per_op[i]) continue;
        const size_t b = std::min(i, s.per_op.size() - 1);
        s.per_op[b] += d.per_op[i];
      }
    }
    return s;
  }
  std::vector<Tracepoint> trace() const {
    std::vector<gpuos_tracepoint> raw(cfg_.trace_capacity ? cfg_.trace_capacity : 1);
    uint64_t n = 0;
    gpuos_trace_snapshot(dev_, raw.data(), raw.size(), &n);
    std::vector<Tracepoint> out;
    out.reserve(n + inline_trace_.size());
    for (uint64_t i = 0; i < n; ++i) {
      Tracepoint t;
      t.seq = raw[i].seq;
      t.op_id = raw[i].op_id;
      t.worker = raw[i].worker;
      t.enqueue_ns = raw[i].enqueue_ns;
      t.dequeue_ns = raw[i].dequeue_ns;
      t.exec_ns = raw[i].exec_ns;
      t.version = raw[i].version;
      out.push_back(t);
    }
    {
      std::lock_guard<std::mutex> lk(trace_mu_);
      out.insert(out.end(), inline_trace_.begin(), inline_trace_.end());
    }
    std::stable_sort(out.begin(), out.end(),
                     [](const Tracepoint& a, const Tracepoint& b) { return a.enqueue_ns < b.enqueue_ns; });
    if (out.size() > cfg_.trace_capacity) out.erase(out.begin(), out.end() - static_cast<long>(cfg_.trace_capacity));
    return out;
  }

  bool worker_alive() const { return gpuos_dev_alive(dev_) != 0; }
  size_t num_workers() const {
    uint32_t n = 0;
    gpuos_dev_num_workers(dev_, &n);
    return n;
  }
  uint64_t canary_hits() const {
    gpuos_dev_stats d{};
    return gpuos_dev_get_stats(dev_, &d) == 0 ? d.canary_hits : 0;
  }
  void set_yield_every(uint64_t n) { gpuos_set_yield_every(dev_, n); }
  bool stopped() const { return stopped_; }
  size_t pending_composites() const { return chain_.size(); }
  gpuos_dev* device() const { return dev_; }
  const RuntimeConfig& config() const { return cfg_; }

  /// Drain, stop the worker kernel, release all buffers; idempotent.
  void shutdown() {
    NvtxRange nvtx_("gpuos::shutdown");
    if (stopped_) return;
    flush_chain();
    wait_all();
    stopped_ = true;
    cells_->pause(1);  // stays paused: every committed task completed above
    gpuos_dev_stop(dev_);
    pool_->clear();
  }

  /// Benchmark hook: drain and stop the worker kernel, then relaunch it (the
  /// ring, table and buffers persist).  Lets a timed step bracket one whole
  /// kernel lifetime with CUDA events.
  void restart_workers() {
    wait_all();
    cells_->pause(1);
    const int rc = gpuos_dev_stop(dev_);
    const int rc2 = rc ? rc : gpuos_dev_start(dev_);
    cells_->pause(-1);
    check_abi(rc, "stop");
    check_abi(rc2, "start");
  }

 private:
  static RuntimeConfig normalize(RuntimeConfig cfg) {
    if (cfg.max_chain == 0) cfg.max_chain = 1;
    if (cfg.table_slots < kFirstInjectedId + 1) cfg.table_slots = kFirstInjectedId + 1;
    return cfg;
  }

  // The composite slot (id 31) holds an identity program until fusion lands.
  static Bytecode composite_placeholder() { return {{OpCode::LoadIn, 0, 0.0}, {OpCode::StoreOut, 0, 0.0}}; }

  static ErrorCode validate(std::span<const TensorView> inputs, const TensorView& output,
                            std::span<const double> scalars) {
    if (inputs.size() > kMaxInputs || scalars.size() > kMaxScalars) return ErrorCode::ArityError;
    if (output.buffer == kInvalidBuffer) return ErrorCode::InvalidBuffer;
    if (output.strides.size() != output.shape.size()) return ErrorCode::IncompatibleShapes;
    for (const TensorView& v : inputs) {
      if (v.buffer == kInvalidBuffer) return ErrorCode::InvalidBuffer;
      if (v.strides.size() != v.shape.size()) return ErrorCode::IncompatibleShapes;
    }
    return ErrorCode::Ok;
  }

  static uint64_t work_elements(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output) {
    if (op_id < kNumBuiltinOps) {
      switch (static_cast<OpKind>(op_id)) {
        case OpKind::ReduceSum: case OpKind::ReduceMax: case OpKind::ReduceMin:
          return inputs.empty() ? 0 : static_cast<uint64_t>(inputs[0].numel());
        case OpKind::Sdpa:
          return inputs.size() >= 2 ? static_cast<uint64_t>(inputs[1].numel()) : 0;
        case OpKind::KvAppend:
          return inputs.size() >= 2 ? static_cast<uint64_t>(inputs[0].numel() + inputs[1].numel()) : 0;
        default: break;
      }
    }
    return static_cast<uint64_t>(output.numel());
  }

  /// Routing filter (runtime.hpp:503-538), with matmul/vecmat queued when
  /// cfg_.queue_matmul (their own 256 cap then applies on the worker).
  bool eligible(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output) const {
    bool kind_ok = false;
    if (op_id >= kFirstInjectedId) {
      kind_ok = op_id <= UINT32_MAX && modules_by_id_.count(static_cast<uint32_t>(op_id)) != 0;
    } else if (op_id < kNumBuiltinOps) {
      switch (static_cast<OpKind>(op_id)) {
        case OpKind::Sdpa:
          kind_ok = inputs.size() >= 2 && inputs[1].rank() == 3 && inputs[1].shape[1] <= cfg_.max_sdpa_context;
          break;
        case OpKind::MatMulSmall: case OpKind::VecMat:
          kind_ok = cfg_.queue_matmul;
          break;
        default:
          kind_ok = true;
      }
    }
    return kind_ok && work_elements(op_id, inputs, output) <= cfg_.max_elements;
  }

  // Resolve a view to the device descriptor (BoundView's checks move here,
  // reported by the body at the reference's bind point).
  bool bind(const TensorView& v, gpuos_view* out) const {
    if (v.rank() > GPUOS_MAX_RANK) return false;
    out->dtype = static_cast<uint8_t>(v.dtype);
    out->rank = static_cast<uint8_t>(v.rank());
    out->status = GPUOS_VIEW_OK;
    out->reserved = 0;
    out->buffer_lo = static_cast<uint32_t>(v.buffer);
    out->addr = 0;
    int64_t lo = v.offset, hi = v.offset, n = 1;
    for (size_t d = 0; d < v.rank(); ++d) {
      const int64_t e = v.shape[d], s = v.strides[d];
      if (e < 0 || e > INT32_MAX || s > INT32_MAX || s < INT32_MIN) return false;
      out->extents[d] = static_cast<int32_t>(e);
      out->strides[d] = static_cast<int32_t>(s);
      n *= e;
      if (e > 0) (s > 0 ? hi : lo) += (e - 1) * s;
    }
    for (size_t d = v.rank(); d < GPUOS_MAX_RANK; ++d) out->extents[d] = out->strides[d] = 0;
    const BufferPool::Buffer* b = pool_->find(v.buffer);
    if (!b) {
      out->status = GPUOS_VIEW_UNKNOWN_BUFFER;
    } else if (b->dtype != v.dtype) {
      out->status = GPUOS_VIEW_DTYPE_VS_BUFFER;
    } else if (n > 0 && (lo < 0 || hi >= static_cast<int64_t>(b->length))) {
      out->status = GPUOS_VIEW_OUT_OF_BOUNDS;
    } else {
      out->addr = reinterpret_cast<uint64_t>(static_cast<char*>(b->data) + v.offset * static_cast<int64_t>(dtype_width(v.dtype)));
    }
    return true;
  }

  // ---- fusion machinery ----
  struct ChainStep {
    uint64_t op_id;
    std::vector<TensorView> inputs;
    TensorView output;
    uint32_t cell;
    uint64_t id;
  };

  /// Structural screen (runtime.hpp:643-673).
  bool chainable(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output) const {
    if (output.dtype != DType::F32 && output.dtype != DType::F64) return false;
    for (const TensorView& v : inputs)
      if (v.dtype != output.dtype) return false;
    size_t want = 0;
    if (op_id >= kFirstInjectedId) {
      const auto it = modules_by_id_.find(static_cast<uint32_t>(op_id));
      if (it == modules_by_id_.end()) return false;
      want = static_cast<size_t>(it->second->signature.arity);
      if (it->second->signature.dtype != output.dtype) return false;
    } else {
      switch (static_cast<OpKind>(op_id)) {
        case OpKind::Add: case OpKind::Mul: want = 2; break;
        case OpKind::Relu: case OpKind::Gelu: want = 1; break;
        default: return false;
      }
      if (table_->latest_entry(op_id).status != OpStatus::Active) return false;
    }
    return inputs.size() == want;
  }

  /// Aliasing rules of runtime.hpp:678-729.
  bool chain_try_append(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
                        uint32_t cell, uint64_t id) {
    if (!chain_.empty()) {
      const TensorView& head = chain_.front().output;
      if (output.dtype != head.dtype || !(output.shape == head.shape)) return false;
    }
    size_t fresh = 0;
    for (const TensorView& in : inputs) {
      bool inter = false, mismatch = false;
      for (const ChainStep& st : chain_) {
        if (in.buffer != st.output.buffer) continue;
        if (in.same_layout(st.output)) inter = true;
        else mismatch = true;
      }
      if (mismatch && !inter) return false;
      if (inter) continue;
      bool known = false;
      for (const TensorView& e : chain_externals_)
        if (in.same_layout(e)) known = true;
      if (!known) ++fresh;
    }
    if (chain_externals_.size() + fresh > kMaxInputs) return false;
    for (const TensorView& e : chain_externals_)
      if (output.buffer == e.buffer) return false;  // would invalidate a folded read
    for (const ChainStep& st : chain_)
      if (output.buffer == st.output.buffer && !output.same_layout(st.output)) return false;
    for (const TensorView& in : inputs) {
      bool inter = false, known = false;
      for (const ChainStep& st : chain_)
        if (in.same_layout(st.output)) inter = true;
      if (inter) continue;
      for (const TensorView& e : chain_externals_)
        if (in.same_layout(e)) known = true;
      if (!known) chain_externals_.push_back(in);
    }
    chain_.push_back(ChainStep{op_id, std::vector<TensorView>(inputs.begin(), inputs.end()), output, cell, id});
    return true;
  }

  /// Builtins re-expressed in the kernels' evaluation order (runtime.hpp:734-762).
  ExprPtr step_ast(const ChainStep& st) const {
    if (st.op_id >= kFirstInjectedId) return clone(*modules_by_id_.at(static_cast<uint32_t>(st.op_id))->folded_ast);
    switch (static_cast<OpKind>(st.op_id)) {
      case OpKind::Add: return make_binary(ExprKind::Add, make_in(0), make_in(1));
      case OpKind::Mul: return make_binary(ExprKind::Mul, make_in(0), make_in(1));
      case OpKind::Relu: return make_binary(ExprKind::Max, make_in(0), make_const(0.0));
      case OpKind::Gelu: {
        const double c = std::sqrt(2.0 / 3.14159265358979323846);
        ExprPtr x3 = make_binary(
            ExprKind::Mul,
            make_binary(ExprKind::Mul, make_binary(ExprKind::Mul, make_const(0.044715), make_in(0)), make_in(0)),
            make_in(0));
        ExprPtr inner = make_binary(ExprKind::Mul, make_const(c), make_binary(ExprKind::Add, make_in(0), std::move(x3)));
        ExprPtr outer = make_binary(ExprKind::Add, make_const(1.0), make_unary(ExprKind::Tanh, std::move(inner)));
        return make_binary(ExprKind::Mul, make_binary(ExprKind::Mul, make_const(0.5), make_in(0)), std::move(outer));
      }
      default: throw Error(ErrorCode::Internal, "unfusable op in chain");
    }
  }

  bool retained(const ChainStep& st) const { return cells_->use_count(st.cell) > chain_handle_baseline_; }

  void flush_chain() {
    NvtxRange nvtx_("gpuos::flush_chain");
    if (chain_.empty()) return;
    std::vector<ChainStep> steps = std::move(chain_);
    chain_.clear();
    chain_externals_.clear();
    size_t i = 0;
    while (i < steps.size()) {
      size_t j = i;
      while (j + 1 < steps.size() && !retained(steps[j])) ++j;
      publish_segment(steps, i, j, /*blocking=*/j + 1 < steps.size());
      i = j + 1;
    }
  }

  void wait_cell(uint32_t cell, uint64_t id) const {
    for (uint32_t spin = 0;; ++spin) {
      const uint64_t w = __atomic_load_n(cells_->word(cell), __ATOMIC_ACQUIRE);
      if ((w & 0xffu) != 0 && (w >> 16) == (id & detail::CellPool::kSeqMask)) return;
      if (spin > 4096) std::this_thread::yield();
      else __builtin_ia32_pause();
    }
  }

  /// Steps [i..j] as one composite task at the composite id (runtime.hpp:785-908).
  void publish_segment(std::vector<ChainStep>& steps, size_t i, size_t j, bool blocking) {
    if (i == j) {  // a single step publishes as itself
      const ChainStep& st = steps[i];
      route(st.op_id, st.inputs, st.output, {}, st.cell, st.id, true, 0);
      if (blocking) wait_cell(st.cell, st.id);
      return;
    }
    const DType dtype = steps[j].output.dtype;
    std::vector<TensorView> ext;
    std::vector<std::pair<TensorView, ExprPtr>> inter;  // produced within this segment
    ExprPtr cur;
    for (size_t k = i; k <= j; ++k) {
      const ChainStep& st = steps[k];
      const ExprPtr base = step_ast(st);
      cur = rewrite_inputs(*base, [&](int idx) -> ExprPtr {
        const TensorView& v = st.inputs[static_cast<size_t>(idx)];
        for (const auto& [iv, ie] : inter)
          if (v.same_layout(iv)) return clone(*ie);
        for (size_t e = 0; e < ext.size(); ++e)
          if (v.same_layout(ext[e])) return make_in(static_cast<int>(e));
        ext.push_back(v);
        return make_in(static_cast<int>(ext.size() - 1));
      });
      if (k < j) {  // materialization boundary: narrow to the stored dtype
        ExprPtr narrowed = make_narrow(dtype, clone(*cur));
        bool replaced = false;
        for (auto& [iv, ie] : inter)
          if (iv.same_layout(st.output)) {
            ie = std::move(narrowed);
            replaced = true;
            break;
          }
        if (!replaced) inter.emplace_back(st.output, std::move(narrowed));
      }
    }
    auto sequential = [&] {
      for (size_t k = i; k <= j; ++k) execute_inline(steps[k].op_id, steps[k].inputs, steps[k].output, {}, steps[k].cell, steps[k].id);
    };
    if (ext.size() > kMaxInputs) {
      sequential();
      return;
    }
    OperatorSignature sig;
    {
      std::string canon;
      detail::canonical_expr(*cur, canon);
      sig.template_name = "fused_" + canon;
    }
    sig.dtype = dtype;
    sig.arity = static_cast<int>(ext.size());
    const uint64_t h0 = cache_.hits(), m0 = cache_.misses();
    ModulePtr mod;
    try {
      mod = cache_.compile_or_get_ast(sig, [&] { return clone(*cur); });
    } catch (...) {
      sync_cache_counters(h0, m0);
      sequential();  // e.g. deeper than the verifier's stack bound: sequential semantics
      return;
    }
    sync_cache_counters(h0, m0);
    const std::string key = signature_key(sig);
    uint64_t prog = 0;
    if (auto it = composite_programs_.find(key); it != composite_programs_.end()) {
      prog = it->second;
    } else {
      const std::vector<gpuos_instr> img = to_device_program(mod->bytecode);
      check_abi(gpuos_program_upload(dev_, img.data(), static_cast<uint32_t>(img.size()), sig.arity,
                                     static_cast<int>(dtype), &prog),
                "composite program");
      composite_programs_.emplace(key, prog);
    }
    fusion_absorbed_ += j - i;  // j-i+1 steps behind one descriptor
    const ChainStep& last = steps[j];
    uint64_t rec_dev = 0;
    uint64_t* rec = cells_->record(last.cell, &rec_dev);
    rec[0] = j - i;
    for (size_t k = i; k < j; ++k) {
      rec[1 + 2 * (k - i)] = cells_->device_addr(steps[k].cell);
      rec[2 + 2 * (k - i)] = steps[k].id;
    }
    double sc[2];
    std::memcpy(&sc[0], &prog, 8);
    std::memcpy(&sc[1], &rec_dev, 8);
    alignas(64) gpuos_task t;
    build_task(kCompositeOpId, ext, last.output, std::span<const double>(sc, 2), last.cell, last.id,
               GPUOS_FLAG_FUSED_COMPOSITE, &t);
    uint64_t pos = 0;
    if (reserve_with_backpressure(&pos)) {
      gpuos_ring_publish(dev_, pos, &t);
      counters_->inc_committed();
      ++committed_tasks_;
      if (blocking) wait_cell(last.cell, last.id);
      return;
    }
    // queue full: the composite on the conventional path, completed here
    counters_->inc_queue_full_fallback();
    counters_->inc_inline();
    ErrorCode code = ErrorCode::Ok;
    int rc = gpuos_launch_task(dev_, &t, inline_stream_);
    if (rc == 0) rc = gpuos_stream_sync(dev_, inline_stream_);
    if (rc != 0) {
      code = static_cast<ErrorCode>(rc);
    } else {
      const uint64_t w = __atomic_load_n(cells_->word(last.cell), __ATOMIC_ACQUIRE);
      code = (w & 0xffu) == 1 ? ErrorCode::Ok : static_cast<ErrorCode>((w >> 8) & 0xffu);
    }
    if (code != ErrorCode::Ok) counters_->inc_failed();
    counters_->inc_op(kCompositeOpId);
    for (size_t k = i; k <= j; ++k) cells_->complete(steps[k].cell, steps[k].id, code);
  }

  bool build_task(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
                  std::span<const double> scalars, uint32_t cell, uint64_t id, uint16_t flags, gpuos_task* t) const {
    t->pub = 0;
    t->seq = id;
    t->op_id = static_cast<uint32_t>(op_id);
    t->flags = flags;
    t->n_inputs = static_cast<uint8_t>(inputs.size());
    t->n_scalars = static_cast<uint8_t>(scalars.size());
    t->size = static_cast<uint64_t>(output.numel());
    t->done_cell = cells_->device_addr(cell);
    t->enqueue_ns = 0;
    if (fence_on_) {  // fence(): wait on the device for the tasks committed before it
      t->flags |= GPUOS_FLAG_AFTER;
      t->enqueue_ns = fence_target_;
    }
    t->aux = 0;
    t->checksum = 0;
    for (size_t i = 0; i < kMaxScalars; ++i) t->scalars[i] = i < scalars.size() ? scalars[i] : 0.0;
    if (!bind(output, &t->views[0])) return false;
    for (size_t i = 0; i < inputs.size(); ++i)
      if (!bind(inputs[i], &t->views[1 + i])) return false;
    for (size_t i = inputs.size(); i < kMaxInputs; ++i) std::memset(&t->views[1 + i], 0, sizeof(gpuos_view));
    t->reserved2[0] = t->reserved2[1] = 0;
    return true;
  }

  /// Dense fast path (the small-op common case): every operand a contiguous,
  /// in-range view of the output's dtype and shape, at most one scalar.  Goes
  /// straight into the ring's compact slot encoding; returns false (nothing
  /// published) when the call does not qualify or the ring is full.
  // The dense slot is written on this thread (gdev::ring_write_dense, the code
  // gpuos_ring_submit_dense runs inside the library) through the producer
  // view fetched at construction: no library call per task.
  int publish_dense_slot(const gpuos_dense_task& t) {
#ifdef GPUOS_NO_INLINE_PUBLISH
    return gpuos_ring_submit_dense(dev_, &t);
#else
    return gdev::ring_write_dense(ring_, t);
#endif
  }

  bool try_publish_dense(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
                         std::span<const double> scalars, uint32_t cell, uint64_t id, uint16_t flags, bool* full) {
    const size_t rank = output.rank();
    if (scalars.size() > 1 || rank > GPUOS_MAX_RANK || op_id > UINT32_MAX) return false;
    gpuos_dense_task t;
    t.seq = id;
    t.done_cell = cells_->device_addr(cell);
    t.op_id = static_cast<uint32_t>(op_id);
    t.flags = fence_on_ ? static_cast<uint16_t>(flags | GPUOS_FLAG_AFTER) : flags;
    t.wait_target = fence_target_;
    t.n_inputs = static_cast<uint8_t>(inputs.size());
    t.n_scalars = static_cast<uint8_t>(scalars.size());
    t.dtype = static_cast<uint8_t>(output.dtype);
    t.rank = static_cast<uint8_t>(rank);
    std::memset(t.reserved, 0, sizeof(t.reserved));
    int64_t n = 1;
    for (size_t d = 0; d < GPUOS_MAX_RANK; ++d) {
      const int64_t e = d < rank ? output.shape[d] : 0;
      if (e < 0 || e > INT32_MAX) return false;
      t.extents[d] = static_cast<int32_t>(e);
      if (d < rank) n *= e;
    }
    t.size = static_cast<uint64_t>(n);
    t.scalar0 = scalars.empty() ? 0.0 : scalars[0];
    const size_t w = dtype_width(output.dtype);
    for (size_t k = 0; k <= inputs.size(); ++k) {
      const TensorView& v = k == 0 ? output : inputs[k - 1];
      if (v.dtype != output.dtype || v.rank() != rank) return false;
      int64_t acc = 1;
      for (size_t d = rank; d-- > 0;) {
        if (v.shape[d] != output.shape[d] || v.strides[d] != acc) return false;  // exact contiguous strides
        acc *= v.shape[d];
      }
      const BufferPool::Buffer* b = pool_->find(v.buffer);
      if (!b || b->dtype != v.dtype || v.offset < 0 || (n > 0 && v.offset + n > static_cast<int64_t>(b->length)))
        return false;  // the general path reports the bind status
      t.addr[k] = reinterpret_cast<uint64_t>(static_cast<char*>(b->data) + v.offset * static_cast<int64_t>(w));
    }
    for (size_t k = inputs.size() + 1; k <= GPUOS_MAX_INPUTS; ++k) t.addr[k] = 0;
    int rc = publish_dense_slot(t);
    if (rc == static_cast<int>(ErrorCode::QueueFull) && cfg_.queue_full_spin_ns) {
      const uint64_t t0 = monotonic_ns();
      do {
        _mm_pause();
        rc = publish_dense_slot(t);
      } while (rc == static_cast<int>(ErrorCode::QueueFull) && monotonic_ns() - t0 < cfg_.queue_full_spin_ns);
    }
    *full = rc == static_cast<int>(ErrorCode::QueueFull);
    return rc == 0;
  }

  void route(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
             std::span<const double> scalars, uint32_t cell, uint64_t id, bool elig, uint16_t flags) {
    if (elig) {
      bool full = false;
      if (try_publish_dense(op_id, inputs, output, scalars, cell, id, flags, &full)) {
        counters_->inc_committed();
        ++committed_tasks_;
        return;
      }
      if (full) {
        counters_->inc_queue_full_fallback();
        execute_inline(op_id, inputs, output, scalars, cell, id);
        return;
      }
    }
    // Views of rank > 4 or with extents/strides beyond int32 do not fit a
    // slot (the reference spills them, queue.hpp:207-221); they take the
    // conventional path, which reports TooLarge for them.
    alignas(64) gpuos_task t;
    if (elig && op_id <= UINT32_MAX && build_task(op_id, inputs, output, scalars, cell, id, flags, &t)) {
      uint64_t pos = 0;
      if (reserve_with_backpressure(&pos)) {
        gpuos_ring_publish(dev_, pos, &t);
        counters_->inc_committed();
        ++committed_tasks_;
        return;
      }
      counters_->inc_queue_full_fallback();
    }
    execute_inline(op_id, inputs, output, scalars, cell, id);
  }

  bool reserve_with_backpressure(uint64_t* pos) {
    if (gpuos_ring_reserve(dev_, pos) == 0) return true;
    if (!cfg_.queue_full_spin_ns) return false;
    const uint64_t t0 = monotonic_ns();
    do {
      _mm_pause();
      if (gpuos_ring_reserve(dev_, pos) == 0) return true;
    } while (monotonic_ns() - t0 < cfg_.queue_full_spin_ns);
    return false;
  }

  void execute_inline(uint64_t op_id, std::span<const TensorView> inputs, const TensorView& output,
                      std::span<const double> scalars, uint32_t cell, uint64_t id) {
    counters_->inc_inline();
    // after a fence(), a synchronous inline run must not overtake the ring
    // tasks committed before the fence
    if (fence_on_) gpuos_ring_wait_processed(dev_, fence_target_);
    const uint64_t t0 = monotonic_ns();
    ErrorCode code = ErrorCode::Ok;
    if (op_id >= table_->slots()) {
      code = ErrorCode::OutOfRange;
    } else {
      const OperatorEntry e = table_->latest_entry(op_id);
      if (e.status == OpStatus::Empty) code = ErrorCode::NotInstalled;
      else if (e.status == OpStatus::Killed) code = ErrorCode::OperatorKilled;
    }
    if (code == ErrorCode::Ok) {
      // matmuls run uncapped on the conventional path (runtime.hpp:589-594)
      const uint16_t flags = (op_id == static_cast<uint64_t>(OpKind::MatMulSmall) ||
                              op_id == static_cast<uint64_t>(OpKind::VecMat))
                                 ? GPUOS_FLAG_UNCAPPED
                                 : 0;
      alignas(64) gpuos_task t;
      if (!build_task(op_id, inputs, output, scalars, cell, id, flags, &t)) {
        code = ErrorCode::TooLarge;
      } else {
        int rc = gpuos_launch_task(dev_, &t, inline_stream_);
        if (rc == 0) rc = gpuos_stream_sync(dev_, inline_stream_);
        if (rc != 0) {
          code = static_cast<ErrorCode>(rc);
        } else {
          const uint64_t w = __atomic_load_n(cells_->word(cell), __ATOMIC_ACQUIRE);
          code = (w & 0xffu) == 1 ? ErrorCode::Ok : static_cast<ErrorCode>((w >> 8) & 0xffu);
        }
      }
    }
    uint64_t t1 = monotonic_ns();
    if (t1 <= t0) t1 = t0 + 1;
    if (code != ErrorCode::Ok) counters_->inc_failed();
    counters_->inc_op(op_id);
    if (cfg_.telemetry_enabled) {
      Tracepoint tp;
      tp.seq = id;
      tp.op_id = op_id;
      tp.worker = 0xFFFFFFFFu;
      tp.enqueue_ns = t0;
      tp.dequeue_ns = t0;
      tp.exec_ns = t1 - t0;
      tp.version = table_->snapshot_version();
      std::lock_guard<std::mutex> lk(trace_mu_);
      inline_trace_.push_back(tp);
      if (inline_trace_.size() > cfg_.trace_capacity) inline_trace_.erase(inline_trace_.begin());
    }
    cells_->complete(cell, id, code);
  }

  void sync_cache_counters(uint64_t h0, uint64_t m0) {
    for (uint64_t k = cache_.hits() - h0; k > 0; --k) counters_->inc_cache_hit();
    for (uint64_t k = cache_.misses() - m0; k > 0; --k) counters_->inc_cache_miss();
  }

  RuntimeConfig cfg_;
  gpuos_dev* dev_ = nullptr;
  std::unique_ptr<BufferPool> pool_;
  std::unique_ptr<OperatorTable> table_;
  detail::CellPool* cells_ = nullptr;
  std::unique_ptr<Counters> counters_;
  ModuleCache cache_;
  TemplateRegistry registry_ = TemplateRegistry::with_defaults();
  void* inline_stream_ = nullptr;
  bool stopped_ = false;
  bool fusion_on_ = false;
  uint64_t next_id_ = 1;
  uint64_t committed_tasks_ = 0;
  gpuos_ring_view ring_{};  // producer view for the inline dense publisher
  uint64_t fence_target_ = 0;  // committed_tasks_ at the last fence()
  bool fence_on_ = false;
  uint64_t next_injected_id_ = kFirstInjectedId;
  std::unordered_map<uint32_t, ModulePtr> modules_by_id_;
  gpuos_inject_stats last_inject_{};
  // native promotion: op id -> jit slot, slot -> signature key, key -> object
  std::unordered_map<uint32_t, uint32_t> native_slot_;
  std::map<uint32_t, std::string> native_obj_;
  std::unordered_map<std::string, std::string> native_cache_;
  NativeStats last_native_{};
  std::vector<ChainStep> chain_;
  std::vector<TensorView> chain_externals_;
  uint64_t fusion_absorbed_ = 0;
  long chain_handle_baseline_ = 0;  // a step is retained while more handles than this reference it
  std::unordered_map<std::string, uint64_t> composite_programs_;  // fused signature -> device program

  static std::string native_symbol(const std::string& key) {
    uint64_t h = 1469598103934665603ull;  // FNV-1a of the signature key
    for (const unsigned char ch : key) h = (h ^ ch) * 1099511628211ull;
    char buf[40];
    std::snprintf(buf, sizeof(buf), "gpuos_native_ptr_%016llx", static_cast<unsigned long long>(h));
    return buf;
  }

  /// CUDA C++ for one verified program: the stack machine unrolled into
  /// straight-line fp64 code with exactly the interpreter's operations
  /// (ops_elementwise.cuh run_program), wrapped in jit_body.
  static std::string native_source(const Bytecode& code, int arity, DType dtype, const std::string& key) {
    const std::string sym = native_symbol(key);
    const std::string tag = sym.substr(std::string("gpuos_native_ptr_").size());
    std::string body;
    std::vector<std::string> st;
    int tmp = 0;
    char line[160];
    auto fresh = [&]() { return "t" + std::to_string(tmp++); };
    for (const Instr& in : code) {
      std::string r;
      switch (in.op) {
        case OpCode::PushConst: {
          uint64_t bits;
          std::memcpy(&bits, &in.value, 8);
          r = fresh();
          std::snprintf(line, sizeof(line), "    const double %s = __longlong_as_double(0x%016llxll);\n", r.c_str(),
                        static_cast<unsigned long long>(bits));
          break;
        }
        case OpCode::LoadIn:
          r = fresh();
          std::snprintf(line, sizeof(line), "    const double %s = v[%d];\n", r.c_str(), in.k);
          break;
        case OpCode::StoreOut:
          std::snprintf(line, sizeof(line), "    return %s;\n", st.back().c_str());
          body += line;
          continue;
        case OpCode::Add: case OpCode::Sub: case OpCode::Mul: case OpCode::Div: case OpCode::Max: case OpCode::Min: {
          const std::string b = st.back();
          st.pop_back();
          const std::string a = st.back();
          st.pop_back();
          r = fresh();
          const char* fn = in.op == OpCode::Add ? "__dadd_rn" : in.op == OpCode::Sub ? "__dsub_rn"
                         : in.op == OpCode::Mul ? "__dmul_rn" : "__ddiv_rn";
          if (in.op == OpCode::Max)
            std::snprintf(line, sizeof(line), "    const double %s = %s < %s ? %s : %s;\n", r.c_str(), a.c_str(), b.c_str(),
                          b.c_str(), a.c_str());
          else if (in.op == OpCode::Min)
            std::snprintf(line, sizeof(line), "    const double %s = %s < %s ? %s : %s;\n", r.c_str(), b.c_str(), a.c_str(),
                          b.c_str(), a.c_str());
          else
            std::snprintf(line, sizeof(line), "    const double %s = %s(%s, %s);\n", r.c_str(), fn, a.c_str(), b.c_str());
          break;
        }
        default: {  // unary
          const std::string a = st.back();
          st.pop_back();
          r = fresh();
          switch (in.op) {
            case OpCode::Neg: std::snprintf(line, sizeof(line), "    const double %s = -%s;\n", r.c_str(), a.c_str()); break;
            case OpCode::Exp: std::snprintf(line, sizeof(line), "    const double %s = exp(%s);\n", r.c_str(), a.c_str()); break;
            case OpCode::Tanh: std::snprintf(line, sizeof(line), "    const double %s = tanh(%s);\n", r.c_str(), a.c_str()); break;
            case OpCode::Abs: std::snprintf(line, sizeof(line), "    const double %s = fabs(%s);\n", r.c_str(), a.c_str()); break;
            case OpCode::Sqrt: std::snprintf(line, sizeof(line), "    const double %s = __dsqrt_rn(%s);\n", r.c_str(), a.c_str()); break;
            default:  // Narrow
              std::snprintf(line, sizeof(line), "    const double %s = narrow_any(%d, %s);\n", r.c_str(), in.k, a.c_str());
          }
        }
      }
      body += line;
      st.push_back(r);
    }
    std::string src;
    src += "// generated by gpuos::Runtime::promote_native for signature: " + key + "\n";
    src += "#include \"ops_elementwise.cuh\"\n";
    src += "namespace gdev {\nstruct NativeF_" + tag + " {\n  static constexpr int A = " + std::to_string(arity) +
           ";\n  __device__ __forceinline__ double operator()(const double* v) const {\n    (void)v;\n" + body +
           "  }\n};\n}  // namespace gdev\n";
    src += "extern \"C\" __device__ __noinline__ int gpuos_native_op_" + tag +
           "(const gpuos_task* t, const gdev::Ctx* c) {\n  return gdev::jit_body<gdev::NativeF_" + tag + ", " +
           std::to_string(static_cast<int>(dtype)) + ">(t, c);\n}\n";
    src += "extern \"C\" __device__ gdev::OpFn " + sym + " = gpuos_native_op_" + tag + ";\n";
    return src;
  }
  mutable std::mutex trace_mu_;
  std::vector<Tracepoint> inline_trace_;
};

}  // namespace gpuos
