// The persistent sm_100a worker kernel (reference Executor, executor.hpp:45-278,
// re-designed as one resident CTA per SM with warp-specialised stages), the
// module jump table, and the standalone per-task kernels of the conventional
// path (execute_inline, runtime.hpp:567-619 == baseline (a): one
// cudaLaunchKernel per task).
//
// Claim protocol (queue.hpp:179-261 restated for PCIe; ring_format.h):
//   * the fetcher warp takes tickets with atomicAdd on the HBM claim cursor
//     (one, or a batch of four under backlog); tickets are FIFO, so the
//     shutdown sentinel drains all earlier work (executor.hpp:178-184).
//   * it polls the 128-byte slots in mapped pinned memory with one warp-wide
//     read; publication = word 0 == pos+1, torn reads fail a checksum
//     (queue.hpp:249-251); extended descriptors add one read of their
//     extension record.
//   * it frees the slot (word 0 = pos + capacity, queue.hpp:248), snapshots the
//     table version with the publish-then-revalidate epoch protocol
//     (executor.hpp:133-141), resolves the op in the bank of that version with
//     the generation canary (executor.hpp:197-212), and hands the task to an
//     executor group through a shared-memory buffer.
//   * the executor group calls the body through the device jump table; the
//     completer warp posts the completion word with a system-scope store
//     after a gpu-scope release fence, and the per-worker processed count.
#if defined(GPUOS_LAT_STAMPS) || defined(GPUOS_FETCH_PROF)
#include <cstdio>
#endif
#include "dev_common.cuh"
#include "dev_state.h"
#include "gpuos_ring_format.h"
#include "ops_elementwise.cuh"
#include "ops_linalg.cuh"
#include "ops_rowwise.cuh"

namespace gdev {

__device__ __noinline__ int op_killed(const gpuos_task*, const Ctx*) { return GPUOS_OPERATOR_KILLED; }
__device__ __noinline__ int op_missing(const gpuos_task*, const Ctx*) { return GPUOS_NOT_INSTALLED; }

// Module jump table: kind -> device function.  Builtin kinds equal their
// reference op ids (ops.hpp:31-48).
__device__ OpFn g_kind_fns[kNumKinds] = {
    op_add, op_mul, op_relu, op_gelu, op_softmax, op_layernorm, op_reduce_sum, op_reduce_max,
    op_reduce_min, op_matmul, op_vecmat, op_sdpa, op_rope, op_kv_append,
    // 14..63 unused
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing,
    // 64: injected program, 65: killed stub
    op_program, op_killed,
    // 66..79 unused
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing, op_missing,
    op_missing, op_missing, op_missing, op_missing, op_missing, op_missing};

struct SharedCtl {
  uint64_t pos;
  uint64_t version;
  uint64_t aux;
  uint64_t t_deq;
  uint64_t t_ticket;
  uint64_t t_seen;
  uint64_t t_fenced;     // executor group woke for this task
  uint64_t t_end;        // body finished (executor group)
  uint64_t yield_every;  // live knobs sampled by the fetcher with the slot read
  uint32_t trace_on;
  uint32_t kind;
  int32_t code;
  uint32_t exit;
  uint32_t plan;  // kPlanDenseSame etc. (dev_common.cuh)
  uint16_t part, nparts;  // this buffer's share of its task (both groups run one task when idle)
  uint32_t partial;       // 1: not the task's last part -- the completer posts nothing
  uint32_t compact;       // 1: the descriptor is still the raw compact slot in braw[b] (executors expand it)
};

constexpr uint32_t kCtlStride = 112;
static_assert(sizeof(SharedCtl) <= kCtlStride, "SharedCtl must fit its stride");

// Worker CTA shape (warp-specialised pipeline):
//   warp 0      fetcher   : claim tickets -> PCIe slot read -> stage -> resolve
//   warps 1..4  executor group 0 (128 threads)   } two tasks execute at once,
//   warps 5..8  executor group 1 (128 threads)   } so one SM keeps ~2 tasks of
//                                                   HBM traffic in flight
//   warp 9      completer : output fence -> completion word -> counters
// Tasks flow through kBufs shared buffers in ticket order: task k uses buffer
// k % kBufs and executor group k % 2; the completer retires them in order.
constexpr int kGroups = 2;
constexpr int kGroupThreads = 128;
constexpr int kWorkerThreads = 32 + kGroups * kGroupThreads + 32;
constexpr int kWorkerRegs = 112;  // __maxnreg__ below; the inline dense path spills at 96
// The resident worker and one standalone task kernel (8 warps x <=80
// registers) must fit together (the inline fallback runs while the worker is
// resident).  Warps are dealt round-robin to the four SM sub-partitions, each
// with a quarter of the register file, so the bound is per sub-partition: the
// one holding three worker warps and two task-kernel warps.  (At 128 registers
// the task kernel could not co-reside and the inline fallback deadlocked.)
static_assert(((kWorkerThreads / 32 + 3) / 4) * kWorkerRegs * 32 + 2 * 80 * 32 <= 65536 / 4,
              "worker + task kernel exceed a sub-partition's register file");
constexpr int kCompleterWarp = 1 + kGroups * kGroupThreads / 32;
constexpr int kBufs = 8;
// Named barriers: 0 = whole CTA, 1+g = executor group g (task bodies),
// FULL[b] = 3+b (3..10): fetcher arrives, group waits (32 + 128).
// DONE[b] and EMPTY[b] are shared-memory mbarriers (count 1): the group's
// thread 0 arrives on DONE after its group barrier, the completer arrives on
// EMPTY; phase parity = lap & 1.  mbarriers can be tested without blocking,
// so the completer retires every consecutive finished buffer behind one
// release fence.
constexpr int kBarFull = 3;
constexpr int kFullCount = 32 + kGroupThreads;
constexpr int kMaxBatch = 4;  // tickets claimed per atomic / slots per warp-wide read
constexpr uint64_t kSplitMin = 2048;  // output elements below which an idle split is not worth it
constexpr uint32_t kTmemCols = 256;  // 128 per executor group; the rest stays free for standalone kernels
constexpr int kBarExecExit = 15;  // both executor groups, before TMEM is released
// Per-CTA cache of resolved table entries, tagged with the version they were
// resolved under: an entry of version v is immutable while v is current
// (the host rewrites a bank only after every epoch moved past it), so a tag
// hit needs no HBM lookup.
constexpr int kEntryCache = 64;
struct CachedEntry {
  uint64_t version;  // kQuiescent = invalid
  uint64_t aux;
  uint32_t op_id;
  uint32_t kind;
  int32_t code;
  uint32_t pad;
};
static_assert(sizeof(CachedEntry) == 32, "cache entry is 32 bytes");

// Constant per generation: read once from DevState at kernel start into the
// shared header (the fetcher reads it from there: in registers it pushed the
// fetcher's loop past the register budget into local-memory spills)
struct WConst {
  const char* ring;
  const char* ext;
  uint64_t mask, cap;
  const uint64_t* host_tail;
  uint64_t* host_done;
  uint64_t* host_claimed;
  uint64_t* host_epoch;
  uint64_t* dev_epoch;
  TableEntry* bank[2];
  uint32_t table_slots, spin_iterations, backoff_max_exp, num_workers;
};

// Shared header (kHeaderBytes): tasks | ctls | raw slot staging | counters | entry cache.
struct WorkerHeader {
  gpuos_task task[kBufs];
  SharedCtl ctl[kBufs];
  uint64_t raw[kMaxBatch][kSlotWords];  // slots as read, before expansion
  uint64_t braw[kBufs][kSlotWords];     // compact slot of buffer b, expanded by its executor group
  uint64_t done;                        // tasks completed by this CTA (all generations)
  uint64_t claimed;                     // tickets claimed by this CTA (all generations)
  uint64_t mbar[kGroups];               // per-group tensor-core completion barriers
  uint64_t done_bar[kBufs];             // DONE[b]: group -> completer
  uint64_t empty_bar[kBufs];            // EMPTY[b]: completer -> fetcher
  uint32_t mma_phase[kGroups];
  uint32_t tmem_base;                   // kTmemCols columns, kTmemCols/kGroups per group
  uint32_t pad_;
  CachedEntry cache[kEntryCache];
  WConst kc;
#ifdef GPUOS_LAT_STAMPS
  long long dbg[16];  // latency bisection (debug builds only)
#endif
};
static_assert(sizeof(WorkerHeader) <= kHeaderBytes, "worker header overflows");

#ifdef GPUOS_LAT_STAMPS
#define LAT_STAMP(i) (H->dbg[i] = clock64())
#else
#define LAT_STAMP(i) ((void)0)
#endif
// Fetcher hand-off profile (debug builds, make fetch-prof): lane 0 sums the
// clock64 cycles of each hand-off segment; CTAs 0..3 print the means at exit.
#ifdef GPUOS_FETCH_PROF
#define FPROF_DECL long long fp_t = 0, fp_sum[6] = {0, 0, 0, 0, 0, 0}, fp_n = 0;
#define FPROF_MARK(i)                   \
  do {                                  \
    if (lane == 0) {                    \
      const long long now_ = clock64(); \
      if ((i) > 0) fp_sum[(i) - 1] += now_ - fp_t; \
      fp_t = now_;                      \
    }                                   \
  } while (0)
#define FPROF_COUNT() (fp_n += (lane == 0))
#define FPROF_PRINT()                                                                                             \
  do {                                                                                                            \
    if (lane == 0 && w < 4 && fp_n)                                                                               \
      printf("FPROF cta %u tasks %lld cycles/task: buffer %lld expand %lld slot+ctl %lld resolve %lld arrive %lld\n", \
             w, fp_n, fp_sum[0] / fp_n, fp_sum[1] / fp_n, fp_sum[2] / fp_n, fp_sum[3] / fp_n, fp_sum[4] / fp_n);   \
  } while (0)
#else
#define FPROF_DECL
#define FPROF_MARK(i) ((void)0)
#define FPROF_COUNT() ((void)0)
#define FPROF_PRINT() ((void)0)
#endif

// Barrier ids must be immediates where possible (a register id makes ptxas
// reserve all 16); the per-buffer families dispatch over constants.
template <int ID>
__device__ __forceinline__ void bar_sync(int n) {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
template <int ID>
__device__ __forceinline__ void bar_arrive(int n) {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "r"(n) : "memory");
}
template <int BASE, int N>
__device__ __forceinline__ void buf_sync(int b) {
  switch (b) {
    case 0: bar_sync<BASE>(N); break;
    case 1: bar_sync<BASE + 1>(N); break;
    case 2: bar_sync<BASE + 2>(N); break;
    case 3: bar_sync<BASE + 3>(N); break;
    case 4: bar_sync<BASE + 4>(N); break;
    case 5: bar_sync<BASE + 5>(N); break;
    case 6: bar_sync<BASE + 6>(N); break;
    default: bar_sync<BASE + 7>(N); break;
  }
}
template <int BASE, int N>
__device__ __forceinline__ void buf_arrive(int b) {
  switch (b) {
    case 0: bar_arrive<BASE>(N); break;
    case 1: bar_arrive<BASE + 1>(N); break;
    case 2: bar_arrive<BASE + 2>(N); break;
    case 3: bar_arrive<BASE + 3>(N); break;
    case 4: bar_arrive<BASE + 4>(N); break;
    case 5: bar_arrive<BASE + 5>(N); break;
    case 6: bar_arrive<BASE + 6>(N); break;
    default: bar_arrive<BASE + 7>(N); break;
  }
}
static_assert(kBufs == 8 && kBarFull + kBufs <= 15, "buf_sync/buf_arrive dispatch eight buffers below barrier 15");

// Shared-memory mbarrier arrive (release.cta) / non-blocking parity test.
__device__ __forceinline__ void mbar_arrive1(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(mbar))
               : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* mbar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"((uint32_t)__cvta_generic_to_shared(mbar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}



// Publish-then-revalidate (executor.hpp:133-141): the epoch slot holds the
// version dispatched under before any bank is read.
__device__ __forceinline__ uint64_t stable_snapshot(DevState* S, const WConst& K, uint32_t w, uint64_t v) {
  for (;;) {
    st_relaxed_gpu(&K.dev_epoch[w], v);
    st_relaxed_sys(&K.host_epoch[w], v);
    fence_sc_sys();
    const uint64_t now = ld_acquire_gpu(&S->version);
    if (now == v) return v;
    v = now;
  }
}

__device__ __forceinline__ void quiesce(const WConst& K, uint32_t w) {
  st_relaxed_gpu(&K.dev_epoch[w], kQuiescent);
  st_relaxed_sys(&K.host_epoch[w], kQuiescent);
}

__device__ __forceinline__ TableEntry load_entry(const TableEntry* e) {
  uint64_t a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(e) : "memory");
  TableEntry r;
  r.kind = (uint16_t)(a & 0xffff);
  r.status = (uint8_t)((a >> 16) & 0xff);
  r.aux = b;
  return r;
}

// Host-visible per-worker counts, written only by fetcher lane 0 (single
// writer, so the posted writes stay monotone on the host).
struct Mirror {
  uint64_t flushed_claimed = 0, flushed_done = 0;
};
__device__ __forceinline__ void flush_mirror(const WConst& K, uint32_t w, Mirror& m, uint64_t claimed,
                                             uint64_t done) {
  if (claimed != m.flushed_claimed) {
    st_relaxed_sys(&K.host_claimed[w], claimed);  // claimed before done: head >= processed
    m.flushed_claimed = claimed;
  }
  if (done != m.flushed_done) {
    st_relaxed_sys(&K.host_done[w], done);
    m.flushed_done = done;
  }
}

// Resolve op -> (kind, aux, code) under version `ver` (optable.hpp:114-124 +
// the generation canary, executor.hpp:197-212).  Lane 0 only.
__device__ __forceinline__ void resolve(DevState* S, const WConst& K, uint32_t w, WorkerHeader* H, uint32_t op,
                                        uint64_t& ver, uint64_t& my_epoch, SharedCtl* ctl) {
  if (op >= K.table_slots) {
    ctl->code = GPUOS_OUT_OF_RANGE;
    ctl->kind = GPUOS_KIND_KILLED;
    ctl->aux = 0;
    return;
  }
  CachedEntry* ce = &H->cache[op % kEntryCache];
  if (ce->version == ver && ce->op_id == op) {
    ctl->code = ce->code;
    ctl->kind = ce->kind;
    ctl->aux = ce->aux;
    return;
  }
  int code = GPUOS_OK;
  TableEntry e;
  e.kind = 0;
  e.aux = 0;
  for (int retry = 0;; ++retry) {
    e = load_entry(&K.bank[ver & 1][op]);
    const uint64_t gen = ld_relaxed_gpu(&S->bank_gen[ver & 1]);
    code = e.status == 1 ? GPUOS_OK : (e.status == 2 ? GPUOS_OPERATOR_KILLED : GPUOS_NOT_INSTALLED);
    // canary: an entry must carry the generation of its version's bank
    if (code == GPUOS_OK && gen != ver && retry < 4) {
      atomicAdd((unsigned long long*)&S->canary_hits, 1ull);
      ver = stable_snapshot(S, K, w, ld_acquire_gpu(&S->version));
      my_epoch = ver;
      continue;
    }
    break;
  }
  const uint32_t kind = (e.kind < kNumKinds || (e.kind >= kJitKindBase && e.kind < kJitKindBase + kJitSlots))
                            ? e.kind
                            : (uint32_t)GPUOS_KIND_KILLED;
  ctl->code = code;
  ctl->kind = kind;
  ctl->aux = e.aux;
  ce->version = ver;
  ce->op_id = op;
  ce->code = code;
  ce->kind = kind;
  ce->aux = e.aux;
}

// Expand a staged compact slot into the ABI descriptor: lane L (< 24) writes
// task words 2L and 2L+1, exactly the words the host's build_task produced.
__device__ __forceinline__ void expand_compact(const uint64_t* raw, gpuos_task* task, int lane) {
  if (lane >= 24) return;
  uint64_t out[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int wi = 2 * lane + h;
    uint64_t v = 0;
    if (wi < 6) {
      v = raw[wi];
    } else if (wi == 7) {
      v = raw[7];
    } else if (wi == 8) {
      v = raw[15];  // scalars[0]
    } else if (wi >= 16 && wi < 46) {
      const int k = (wi - 16) / 6, f = (wi - 16) % 6;
      const uint32_t n_inputs = (uint32_t)((raw[2] >> 48) & 0xff);
      if ((uint32_t)k <= n_inputs) {
        const uint32_t dtype = (uint32_t)((raw[6] >> 8) & 0xff), rank = (uint32_t)((raw[6] >> 16) & 0xff);
        int32_t ext[4] = {(int32_t)(uint32_t)raw[8], (int32_t)(uint32_t)(raw[8] >> 32), (int32_t)(uint32_t)raw[9],
                          (int32_t)(uint32_t)(raw[9] >> 32)};
        int32_t st[4];
        contiguous_strides4(ext, (int)rank, st);
        switch (f) {
          case 0: v = raw[10 + k]; break;                                         // addr
          case 1: v = raw[8]; break;                                              // extents 0,1
          case 2: v = raw[9]; break;                                              // extents 2,3
          case 3: v = (uint64_t)(uint32_t)st[0] | ((uint64_t)(uint32_t)st[1] << 32); break;
          case 4: v = (uint64_t)(uint32_t)st[2] | ((uint64_t)(uint32_t)st[3] << 32); break;
          default: v = (uint64_t)dtype | ((uint64_t)rank << 8); break;            // status 0, buffer_lo 0
        }
      }
    }
    out[h] = v;
  }
  reinterpret_cast<uint4*>(task)[lane] =
      make_uint4((uint32_t)out[0], (uint32_t)(out[0] >> 32), (uint32_t)out[1], (uint32_t)(out[1] >> 32));
}

// Stage the extension record of an extended slot (task words 16..46): one
// 256-byte read by lanes 0..15, validated against its position-bound checksum.
__device__ __forceinline__ void fetch_ext(DevState* S, const WConst& K, uint64_t pos, gpuos_task* task, int lane) {
  const char* rec = K.ext + (pos & K.mask) * kExtBytes;
  for (;;) {
    uint4 v = make_uint4(0, 0, 0, 0);
    if (lane < 16) v = ld_volatile_v4(rec + 16 * lane);
    const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
    uint64_t part = 0;
    if (lane < 16) {
      part = ring_term(w0, 2 * lane);
      if (lane != 15) part += ring_term(w1, 2 * lane + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    part += ring_term(pos + 1, kExtChecksumSalt);
    const uint64_t chk = shfl64(w1, 15);
    if (part == chk) {
      if (lane < 16) {
        if (lane == 15) v.z = v.w = 0;  // reserved2[1] carried the checksum
        reinterpret_cast<uint4*>(task)[8 + lane] = v;
      }
      __syncwarp();
      return;
    }
    if (lane == 0) atomicAdd((unsigned long long*)&S->torn_reads, 1ull);
  }
}

// Shared state of the fetcher warp (registers, uniform across the warp).
struct Fetcher {
  uint64_t my_epoch = kQuiescent;
  Mirror mir;
  uint32_t k = 0;  // tasks (and exit markers) handed to the executors so far
};

// Hand the next buffer to the executors: wait until the completer released
// it (after its first lap), return its index.
__device__ __forceinline__ int next_buffer(WorkerHeader* H, Fetcher& F) {
  const int b = (int)(F.k % kBufs);
  if (F.k >= (uint32_t)kBufs) mbar_wait(&H->empty_bar[b], ((F.k / kBufs) - 1) & 1);
  return b;
}

// Exit: one marker per executor group (each waits on its own buffers), then
// wait for the completer to release everything in flight, then publish the
// final counts as the single writer of the host mirrors.
__device__ __forceinline__ void fetcher_exit(const WConst& K, uint32_t w, WorkerHeader* H, Fetcher& F, int lane,
                                             bool first_marker_staged) {
  for (int g = first_marker_staged ? 1 : 0; g < kGroups; ++g) {
    const int b = next_buffer(H, F);
    if (lane == 0) {
      H->ctl[b].exit = 1;
      H->ctl[b].partial = 0;
    }
    __syncwarp();
    buf_arrive<kBarFull, kFullCount>(b);
    ++F.k;
  }
  const uint32_t inflight = F.k < (uint32_t)kBufs ? F.k : (uint32_t)kBufs;
  for (uint32_t q = F.k - inflight; q < F.k; ++q) mbar_wait(&H->empty_bar[q % kBufs], (q / kBufs) & 1);
  if (lane == 0) flush_mirror(K, w, F.mir, H->claimed, *(volatile uint64_t*)&H->done);
}

// The fetcher warp's whole life.
//
// Claim: one atomicAdd takes 1 ticket, or kMaxBatch when the device-visible
// tail shows a backlog of more than two tickets per worker (batching then
// costs no latency and cuts PCIe round trips per task by up to 4x).
// Poll: lanes 8j..8j+7 read slot j of the batch (one warp-wide 512-byte read);
// publication = word 0 == pos+1, torn reads fail the slot checksum.  Only
// tickets within two of the highest tail seen on the device read PCIe; the
// rest watch the HBM hint.  Progress: the ticket equal to the hint is always
// near, and its poll carries the producer tail, so every publication
// eventually advances the hint.
__device__ __forceinline__ void fetcher_main(DevState* S, WorkerHeader* H, uint32_t w, int lane) {
  if (lane == 0) {
    WConst& k = H->kc;
    k.ring = S->ring;
    k.ext = S->ext;
    k.mask = S->mask;
    k.cap = S->cap;
    k.host_tail = S->host_tail;
    k.host_done = S->host_done;
    k.host_claimed = S->host_claimed;
    k.host_epoch = S->host_epoch;
    k.dev_epoch = S->dev_epoch;
    k.bank[0] = S->bank[0];
    k.bank[1] = S->bank[1];
    k.table_slots = S->table_slots;
    k.spin_iterations = S->spin_iterations;
    k.backoff_max_exp = S->backoff_max_exp;
    k.num_workers = S->num_workers;
  }
  __syncwarp();
  const WConst& K = H->kc;
  Fetcher F;
  F.mir.flushed_claimed = H->claimed;
  F.mir.flushed_done = H->done;
  uint64_t last_pos = 0, hint_seen = ld_relaxed_gpu(&S->hint);
  const int seg = lane >> 3, sl = lane & 7;
  // claim-ahead: the next batch's tickets are taken while the current batch is
  // handed to the executors, so the HBM atomic's round trip overlaps staging
  uint64_t pre_pos = 0;  // lane 0
  uint32_t pre_nb = 0;   // lane 0
  bool pre = false;      // warp-uniform
  FPROF_DECL
  uint32_t tr_last = 0;  // trace_on as last sampled: phase stamps only when tracing
  for (;;) {
    // ---- claim a batch ----
    uint64_t pos = 0;
    uint32_t nb = 1;
    if (lane == 0) {
      if (pre) {
        pos = pre_pos;
        nb = pre_nb;
      } else {
        while (*(volatile uint32_t*)&S->hold) __nanosleep(2000);
        // Lazy claiming: take a ticket only when the claim cursor is within
        // two of the hint (this fetcher becomes one of the frontier pollers)
        // or the hint says published work lies past the cursor.  Idle workers
        // used to each hold a far ticket and reach it only as the hint crept
        // forward hop by hop; a 32-task burst after idle was picked up in
        // waves 16 us apart (tools/probe/burst_probe).  Now whoever wakes
        // first claims work the hint has already announced.
        for (uint32_t ns = 64;;) {
          const uint64_t cl = ld_relaxed_gpu(&S->claim), hn = ld_relaxed_gpu(&S->hint);
          if ((cl < hn + 2 || ld_relaxed_gpu(&S->stop_pos) != kRunning) && !*(volatile uint32_t*)&S->hold) {
            hint_seen = hn > hint_seen ? hn : hint_seen;
            break;
          }
          // idle: keep the host-visible counts current (wait_all / peek read
          // them; the completer updates H->done after this fetcher's last claim)
          flush_mirror(K, w, F.mir, H->claimed, *(volatile uint64_t*)&H->done);
          __nanosleep(ns);
          if (ns < 1024) ns <<= 1;
        }
        nb = hint_seen > last_pos + 2ull * K.num_workers ? (uint32_t)kMaxBatch : 1u;
        pos = atomicAdd((unsigned long long*)&S->claim, (unsigned long long)nb);
        last_pos = pos + nb - 1;
      }
    }
    pre = false;
    pos = shfl64(pos, 0);
    nb = __shfl_sync(0xffffffffu, nb, 0);
    hint_seen = shfl64(hint_seen, 0);
    uint32_t j = 0;  // next slot of the batch to hand over
    const uint64_t t_ticket = tr_last ? globaltimer() : 0;
    uint32_t spins = 0, expn = 0;
    while (j < nb) {
      // One round of loads, issued back to back: the slots (near tickets
      // only), then the control words on single lanes.  All are relaxed: an
      // acquire would run CCTL.IVALL and drop the executors' L1-resident
      // stacks.  Table entries are L2 loads issued after the version read
      // returned, and the host writes a bank before it publishes the version
      // that selects it, so an entry read under version v sees v's bank.
      // Nearness uses the hint seen by the previous round.
      // Belt and braces for the hint protocol (see the published-slot update
      // below): every 64th idle round a far ticket polls too.
      const bool near = pos + j < hint_seen + 2 || (spins & 63) == 63;
      uint32_t ready = 0;  // consecutive valid slots starting at j
      uint4 v = make_uint4(0, 0, 0, 0);
      uint64_t aux = 0;    // lane 1: version, 2: yield_every, 3: trace_on, 4: tail, 5: stop_pos, 6: hint
      const uint32_t sj = j + (uint32_t)seg;
      const uint64_t spos = pos + sj;
      if (near && sj < nb) v = ld_volatile_v4(K.ring + (spos & K.mask) * kRingSlot + 16 * sl);
      if (near && lane == 4 && pos + nb - 1 >= hint_seen) aux = ld_relaxed_sys(K.host_tail);
      if (lane == 5) aux = ld_relaxed_gpu(&S->stop_pos);
      if (lane == 6) aux = ld_relaxed_gpu(&S->hint);
      if (near && lane == 2) aux = ld_relaxed_gpu(&S->yield_every);
      if (near && lane == 3) aux = *(volatile uint32_t*)&S->trace_on;
      if (near && lane == 1) aux = ld_relaxed_gpu(&S->version);
      const uint64_t sp = shfl64(aux, 5);
      const uint64_t h = shfl64(aux, 6);
      const uint64_t tail = near ? shfl64(aux, 4) : 0;
      if (lane == 0 && tail > h) atomicMax((unsigned long long*)&S->hint, (unsigned long long)tail);
      hint_seen = tail > h ? tail : h;
      if (pos + j > sp) {
        FPROF_PRINT();
        if (lane == 0) {
          quiesce(K, w);
          F.my_epoch = kQuiescent;
        }
        fetcher_exit(K, w, H, F, lane, false);
        return;
      }
      if (near) {
        const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
        uint64_t part = ring_term(w0, 2 * sl);
        if (sl != 3) part += ring_term(w1, 2 * sl + 1);  // word 7 is the checksum
        part += __shfl_xor_sync(0xffffffffu, part, 4);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        const uint64_t pub = shfl64(w0, lane & ~7);
        const uint64_t chk = shfl64(w1, (lane & ~7) + 3);
        const bool valid = sj < nb && pub == spos + 1 && part == chk;
        const bool torn = sj < nb && pub == spos + 1 && part != chk;
        const unsigned vb = __ballot_sync(0xffffffffu, valid && sl == 0);
        const unsigned tb = __ballot_sync(0xffffffffu, torn && sl == 0);
        // consecutive valid segments from segment 0 (bits 0, 8, 16, 24)
        while (ready < (uint32_t)kMaxBatch && (vb >> (8 * ready)) & 1u) ++ready;
        if (ready == 0 && tb != 0 && lane == 0) atomicAdd((unsigned long long*)&S->torn_reads, 1ull);
        if (ready > 0) {
          // A published slot proves the producer tail is past it.  The tail
          // word read in the same round may be older (the two PCIe reads are
          // unordered), so without this the hint could stall below the
          // consumed tickets, leaving no ticket "near" and nobody polling --
          // a stall seen once in a 10^6-task mixed stream.
          const uint64_t past = pos + j + ready;
          if (past > hint_seen) {
            hint_seen = past;
            if (lane == 0) atomicMax((unsigned long long*)&S->hint, (unsigned long long)past);
          }
          const uint32_t tr0 = (uint32_t)shfl64(aux, 3);
          tr_last = tr0;
          const uint64_t t_seen = tr0 ? globaltimer() : 0;
          if (lane == 0) LAT_STAMP(0);
          // No acquire fence: executors read task operands with L2 loads only
          // (coherence rule, dev_common.cuh), issued after this read returned
          // (GPUs do not speculate loads past the validation branch).  An
          // acquire here would run CCTL.IVALL, dropping every warp's L1-resident
          // stack frames along with stale data (measured: +1.5 us per task).
          uint64_t ver = shfl64(aux, 1);
          const uint64_t ye = shfl64(aux, 2);
          const uint32_t tr = (uint32_t)shfl64(aux, 3);
          // stage the raw slots of the valid run
          if ((uint32_t)seg < ready) reinterpret_cast<uint4*>(H->raw[seg])[sl] = v;
          __syncwarp();
          if (j + ready >= nb) {
            // this round consumes the batch: take the next tickets now
            uint32_t took = 0;
            if (lane == 0 && !*(volatile uint32_t*)&S->hold && hint_seen > last_pos) {
              pre_nb = hint_seen > last_pos + 2ull * K.num_workers ? (uint32_t)kMaxBatch : 1u;
              pre_pos = atomicAdd((unsigned long long*)&S->claim, (unsigned long long)pre_nb);
              last_pos = pre_pos + pre_nb - 1;
              took = 1;
            }
            pre = __shfl_sync(0xffffffffu, took, 0) != 0;
          }
          for (uint32_t i = 0; i < ready; ++i) {
            const uint64_t spos = pos + j;
            const uint64_t* raw = H->raw[i];
            FPROF_MARK(0);
            const int b = next_buffer(H, F);
            FPROF_MARK(1);
            gpuos_task* task = &H->task[b];
            SharedCtl* ctl = &H->ctl[b];
            const bool compact = (raw[6] & 0xff) == kFmtCompact;
            // fields the fetcher itself needs, from the raw compact slot
            uint32_t op_id, flags;
            uint64_t tsize, scalar0;
            if (compact) {
              // hand the raw slot over: the executor group expands it (24 of
              // its threads, at wake) -- off the fetcher's per-task path
              if (lane < 8) reinterpret_cast<uint4*>(H->braw[b])[lane] = reinterpret_cast<const uint4*>(raw)[lane];
              op_id = (uint32_t)raw[2];
              flags = (uint32_t)(raw[2] >> 32) & 0xffffu;
              tsize = raw[3];
              scalar0 = raw[15];
            } else {
              if (lane < 8) reinterpret_cast<uint4*>(task)[lane] = reinterpret_cast<const uint4*>(raw)[lane];
              __syncwarp();
              fetch_ext(S, K, spos, task, lane);
            }
            __syncwarp();
            if (!compact) {
              op_id = task->op_id;
              flags = task->flags;
              tsize = task->size;
              scalar0 = (uint64_t)__double_as_longlong(task->scalars[0]);
            }
            FPROF_MARK(2);
            if (lane == 0) LAT_STAMP(1);
            const uint32_t plan = compact ? kPlanDenseSame : plan_task_warp(task, lane);
            bool shutdown = false;
            if (lane == 0) {
              if (flags & GPUOS_FLAG_AFTER) {
                // device-side ordering: every task committed before the fence
                // must have completed (processed is bumped after the
                // completer's release fence, so their outputs are in L2)
                const uint64_t target = compact ? raw[5] : task->enqueue_ns;
                for (uint32_t ns = 32; ld_relaxed_gpu(&S->processed) < target;) {
                  __nanosleep(ns);
                  if (ns < 1024) ns <<= 1;
                }
              }
              // free the slot for the producer's next lap (queue.hpp:248)
              st_relaxed_sys((uint64_t*)(K.ring + (spos & K.mask) * kRingSlot), spos + K.cap);
              const uint64_t claimed = ++H->claimed;
              if ((claimed & 15) == 0) flush_mirror(K, w, F.mir, claimed, *(volatile uint64_t*)&H->done);
              ctl->pos = spos;
              ctl->exit = 0;
              ctl->t_ticket = t_ticket;
              ctl->t_seen = t_seen;
              ctl->yield_every = ye;
              ctl->trace_on = tr;
              ctl->plan = plan;
              ctl->compact = compact ? 1u : 0u;
              LAT_STAMP(2);
              FPROF_MARK(3);
              if (flags & GPUOS_FLAG_SHUTDOWN) {
                atomicMin((unsigned long long*)&S->stop_pos, (unsigned long long)spos);
                quiesce(K, w);
                F.my_epoch = kQuiescent;
                ctl->exit = 1;
                shutdown = true;
              } else {
                if (ver != F.my_epoch) ver = stable_snapshot(S, K, w, ver);
                F.my_epoch = ver;
                resolve(S, K, w, H, op_id, ver, F.my_epoch, ctl);
                if ((flags & GPUOS_FLAG_FUSED_COMPOSITE) && ctl->code == GPUOS_OK) {
                  // fused elementwise chain (runtime.hpp:912-933): the entry at
                  // the composite id gates it; the program rides in scalars[0]
                  ctl->kind = GPUOS_KIND_PROGRAM;
                  ctl->aux = scalar0;
                }
                ctl->version = ver;
                LAT_STAMP(3);
                ctl->t_deq = tr ? globaltimer() : 0;
              }
            }
            FPROF_MARK(4);
            shutdown = __shfl_sync(0xffffffffu, shutdown, 0);
            // Idle split: with nothing else published, a task large enough to
            // split runs on both executor groups -- this buffer takes part 0
            // and the next buffer (the other group's) a copy as part 1.  The
            // completer retires buffers in order, so the task completes once,
            // after both halves.
            const bool split = !shutdown && ready == 1 && nb == 1 && hint_seen <= spos + 1 &&
                               tsize >= kSplitMin;
            if (lane == 0) {
              ctl->part = 0;
              ctl->nparts = split ? 2 : 1;
              ctl->partial = split ? 1u : 0u;
            }
            __syncwarp();
            if (lane == 0) LAT_STAMP(4);
            buf_arrive<kBarFull, kFullCount>(b);
            FPROF_MARK(5);
            FPROF_COUNT();
            ++F.k;
            ++j;
            if (split) {
              const int b2 = next_buffer(H, F);
              if (compact) {
                if (lane < 8) reinterpret_cast<uint4*>(H->braw[b2])[lane] = reinterpret_cast<const uint4*>(H->braw[b])[lane];
              } else if (lane < 24) {
                reinterpret_cast<uint4*>(&H->task[b2])[lane] = reinterpret_cast<const uint4*>(task)[lane];
              }
              if (lane < (int)(sizeof(SharedCtl) / 8))
                reinterpret_cast<uint64_t*>(&H->ctl[b2])[lane] = reinterpret_cast<const uint64_t*>(ctl)[lane];
              __syncwarp();
              if (lane == 0) {
                H->ctl[b2].part = 1;
                H->ctl[b2].partial = 0;
              }
              __syncwarp();
              buf_arrive<kBarFull, kFullCount>(b2);
              ++F.k;
            }
            if (shutdown) {
              // the sentinel's buffer carried the first exit marker
              FPROF_PRINT();
              fetcher_exit(K, w, H, F, lane, true);
              return;
            }
          }
          spins = 0;
          expn = 0;
          continue;
        }
      }
      ++spins;
      if (lane == 0) {
        flush_mirror(K, w, F.mir, H->claimed, *(volatile uint64_t*)&H->done);  // idle: counts for wait_all / peek
        if ((spins & 15) == 0) {
          const uint64_t cur = ld_relaxed_gpu(&S->version);
          if (cur != F.my_epoch) F.my_epoch = stable_snapshot(S, K, w, cur);
          if (spins == K.spin_iterations) atomicAdd((unsigned long long*)&S->stalls, 1ull);
        }
      }
      if (!near) {
        __nanosleep(64u << expn);
        // (a short backoff for tickets near the hint did not narrow the pickup
        // spread of a burst after idle, and polling the producer tail from
        // those tickets congested PCIe: burst pickup 120 us, depth-1 p50 94 us)
        if (expn < K.backoff_max_exp) ++expn;
      }
    }
  }
}

// Completion (runtime.hpp:628-639) by lane 0 of the completer warp.  The
// DONE barrier orders every executor's output writes before the fence; the
// release puts them in L2 (where the host's copy engine reads) before the
// completion word is posted to host memory.
__device__ __forceinline__ void complete_task(DevState* S, uint32_t w, WorkerHeader* H, const gpuos_task* task,
                                              const SharedCtl* ctl, int code, uint64_t t_end, uint64_t& executed,
                                              uint32_t& n_done, uint32_t& n_failed) {
  const uint64_t state = ((uint64_t)(code == GPUOS_OK ? 1 : 2)) | ((uint64_t)(code & 0xff) << 8);
  if ((task->flags & GPUOS_FLAG_FUSED_COMPOSITE) && task->n_scalars > 1) {
    // the chain's earlier steps complete with the composite, in chain order
    // and before the composite's own cell (runtime.hpp:904-908): their (cell,
    // seq) pairs sit in a host-written record (scalars[1]) that the host may
    // reuse once the final cell is posted, so it is read first
    const uint64_t* rec = (const uint64_t*)__double_as_longlong(task->scalars[1]);
    if (rec) {
      const uint64_t nsteps = ld_relaxed_sys(rec);
      for (uint64_t k = 0; k < nsteps && k < GPUOS_MAX_FUSED; ++k) {
        const uint64_t cell = ld_relaxed_sys(rec + 1 + 2 * k), seq = ld_relaxed_sys(rec + 2 + 2 * k);
        st_relaxed_sys((uint64_t*)cell, state | (seq << 16));
      }
      // the composite's own cell is released after the earlier ones
      if (task->done_cell) st_release_sys((uint64_t*)task->done_cell, state | (task->seq << 16));
      goto counted;
    }
  }
  if (task->done_cell) st_relaxed_sys((uint64_t*)task->done_cell, state | (task->seq << 16));
counted:
  *(volatile uint64_t*)&H->done = H->done + 1;
  ++n_done;
  if (code != GPUOS_OK) ++n_failed;
  atomicAdd((unsigned long long*)&S->per_op[task->op_id < 256 ? task->op_id : 255], 1ull);
  if (ctl->trace_on) {
    const uint64_t ticket = atomicAdd((unsigned long long*)&S->trace_head, 1ull);
    TraceRec* r = &S->trace[ticket % S->trace_cap];
    r->stamp = ticket * 2 + 1;
    r->seq = task->seq;
    r->op_id = task->op_id;
    r->worker = w;
    r->enqueue_ns = (task->flags & GPUOS_FLAG_AFTER) ? 0 : task->enqueue_ns;
    r->dequeue_gt = ctl->t_deq;
    r->exec_ns = t_end > ctl->t_deq ? t_end - ctl->t_deq : 1;
    r->version = ctl->version;
    r->t_ticket = ctl->t_ticket;
    r->t_seen = ctl->t_seen;
    r->t_done = globaltimer();
    r->pad = ctl->t_fenced;
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&r->stamp), "l"(ticket * 2 + 2) : "memory");
  }
  ++executed;
  const uint64_t ye = ctl->yield_every;
  if (ye > 0 && executed % ye == 0) __nanosleep(1000);  // yield_every (executor.hpp:190-193)
}

// Guarded devirtualisation of the table's hottest entries.  After resolve()
// has mapped op_id -> kind through the dual-bank table (versioned, aliasable),
// a builtin add or mul over planned dense f32 operands runs inline instead
// of through the function pointer: the indirect call saves and restores ~40
// callee-saved registers through local memory, measured at +2300 cycles on a
// 64-element task (tools/probe/body_bench.cu).  Any other kind, dtype, layout
// arity or alignment takes the jump table.  Returns false when it did not run the task.
struct FAddOrMul {  // one loop for both binary ops (one instantiation, one register budget)
  static constexpr int A = 2;
  static constexpr bool kF32 = true;
  bool mul;
  __device__ __forceinline__ double operator()(const double* v) const {
    return mul ? __dmul_rn(v[0], v[1]) : __dadd_rn(v[0], v[1]);
  }
  __device__ __forceinline__ float f32(const float* v) const { return mul ? __fmul_rn(v[0], v[1]) : __fadd_rn(v[0], v[1]); }
  __device__ __forceinline__ long long i64(const long long* v) const { return mul ? v[0] * v[1] : v[0] + v[1]; }
};
__device__ __forceinline__ bool dense_f32_inline(uint32_t kind, const gpuos_task* t, const Ctx* c) {
  if (kind > GPUOS_OP_MUL || !(c->flags & kPlanDenseSame) || t->views[0].dtype != GPUOS_F32 || t->n_inputs != 2)
    return false;
  const int64_t n = numel(t->views[0]);
  if (n <= 0 || n >= ((int64_t)1 << 31)) return false;
  if ((t->views[0].addr | t->views[1].addr | t->views[2].addr) & 15) return false;
  FAddOrMul f;
  f.mul = kind == GPUOS_OP_MUL;
  ew_dense<GPUOS_F32, FAddOrMul, 4, true>(t, c, n, f);
  return true;
}

// One persistent generation.
extern "C" __global__ void __maxnreg__(kWorkerRegs) gpuos_worker_kernel(DevState* S) {
  extern __shared__ __align__(128) char smem[];
  WorkerHeader* H = reinterpret_cast<WorkerHeader*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t w = blockIdx.x;
  if (tid == 0) {
    // continue the host-visible counts across kernel generations
    H->claimed = ld_relaxed_sys(&S->host_claimed[w]);
    H->done = ld_relaxed_sys(&S->host_done[w]);
  }
  for (int i = tid; i < kEntryCache; i += blockDim.x) {
    H->cache[i].version = kQuiescent;
    H->cache[i].op_id = 0xffffffffu;
  }
  if (tid == 0) {
    for (int g = 0; g < kGroups; ++g) {
      mbar_init(&H->mbar[g], 1);
      H->mma_phase[g] = 0;
    }
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&H->done_bar[b], 1);
      mbar_init(&H->empty_bar[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(&H->tmem_base, kTmemCols);  // owned (and released) by warp 1
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    fetcher_main(S, H, w, lane);
    return;
  }
  if (warp == kCompleterWarp) {
    // ---------------- completer: retires tasks in ticket order ----------------
    // Lane 0 waits for the oldest buffer, then takes every consecutive buffer
    // that is already done; one release fence orders all of their outputs
    // before their completion words (the fence waits for the SM's
    // outstanding writes, so one per run instead of one per task).
    if (lane != 0) return;
    uint64_t executed = 0;
    int exits = 0;
    for (uint32_t k = 0;;) {
      mbar_wait(&H->done_bar[k % kBufs], (k / kBufs) & 1);
      uint32_t n = 1;
      while (n < (uint32_t)kBufs && mbar_test(&H->done_bar[(k + n) % kBufs], ((k + n) / kBufs) & 1)) ++n;
#ifdef GPUOS_COMPLETE_FENCE_SYS
      asm volatile("fence.release.sys;" ::: "memory");
#else
      asm volatile("fence.release.gpu;" ::: "memory");
#endif
      uint32_t n_done = 0, n_failed = 0;
      for (uint32_t i = 0; i < n; ++i, ++k) {
        const int b = (int)(k % kBufs);
        const SharedCtl* ctl = &H->ctl[b];
        if (ctl->exit) {
          ++exits;
          mbar_arrive1(&H->empty_bar[b]);
          continue;
        }
#ifdef GPUOS_LAT_STAMPS
        LAT_STAMP(9);
#endif
        if (!ctl->partial)
          complete_task(S, w, H, &H->task[b], ctl, ctl->code, ctl->t_end, executed, n_done, n_failed);
#ifdef GPUOS_LAT_STAMPS
        if (!ctl->partial) {
          LAT_STAMP(10);
          if (ctl->pos > 40 && ctl->pos % 37 == 0) {
            const long long* d = H->dbg;
            printf("LAT pos %llu size %lld part %d/%d: expand %lld plan+ctl %lld resolve %lld arrive %lld | wake %lld fnload %lld body %lld gsync %lld | done-wake %lld complete %lld\n",
                   (unsigned long long)ctl->pos, (long long)H->task[b].size, ctl->part, ctl->nparts, d[1] - d[0], d[2] - d[1], d[3] - d[2],
                   d[4] - d[3], d[5] - d[4], d[6] - d[5], d[7] - d[6], d[8] - d[7], d[9] - d[8], d[10] - d[9]);
          }
        }
#endif
        mbar_arrive1(&H->empty_bar[b]);
      }
      if (n_done) atomicAdd((unsigned long long*)&S->processed, (unsigned long long)n_done);
      if (n_failed) atomicAdd((unsigned long long*)&S->failed, (unsigned long long)n_failed);
      if (exits == kGroups) return;
    }
  }
  // ---------------- executor group g: tasks g, g+2, g+4, ... ----------------
  const int g = (warp - 1) / (kGroupThreads / 32);
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  const int scratch = ((int)dyn - (int)kHeaderBytes) / kGroups & ~127;
  Ctx ctx;
  ctx.tid = tid - 32 - g * kGroupThreads;
  ctx.nthreads = kGroupThreads;
  ctx.part = 0;
  ctx.nparts = 1;
  ctx.bar_id = 1 + g;
  ctx.smem = smem + kHeaderBytes + g * scratch;
  ctx.smem_bytes = scratch;
  ctx.aux = 0;
  ctx.flags = 0;
  OpFn_* const jit_fns = S->jit_fns;
  ctx.tmem = H->tmem_base + (uint32_t)(g * (kTmemCols / kGroups));
  ctx.mbar = &H->mbar[g];
  ctx.mma_phase = &H->mma_phase[g];
  for (uint32_t k = (uint32_t)g;; k += kGroups) {
    const int b = (int)(k % kBufs);
    buf_sync<kBarFull, kFullCount>(b);
    gpuos_task* task = &H->task[b];
    SharedCtl* ctl = &H->ctl[b];
    if (ctl->exit) {
      if (ctx.tid == 0) mbar_arrive1(&H->done_bar[b]);
      // both groups are past their last tensor-core use: release TMEM
      tc_fence_before();
      bar_sync<kBarExecExit>(kGroups * kGroupThreads);
      tc_fence_after();
      if (warp == 1) tmem_dealloc(H->tmem_base, kTmemCols);
      return;
    }
    if (ctl->compact) {
      // the fetcher handed over the raw compact slot: 24 threads expand it
      if (ctx.tid < 24) expand_compact(H->braw[b], task, ctx.tid);
      group_sync(&ctx);
    }
    const uint64_t t_wake = ctl->trace_on ? globaltimer() : 0;
    if (ctx.tid == 0) LAT_STAMP(5);
    int code = ctl->code;
    if (code == GPUOS_OK) {
      // Rewrite the whole context each task: the body reads it through a
      // pointer to local memory, and lines written long ago have left L1
      // (measured: a field stored at kernel start reloads from L2 at ~330
      // cycles, a field stored this task at ~50).
      ctx.tid = tid - 32 - g * kGroupThreads;
      ctx.nthreads = kGroupThreads;
      ctx.bar_id = 1 + g;
      ctx.smem = smem + kHeaderBytes + g * scratch;
      ctx.smem_bytes = scratch;
      ctx.tmem = H->tmem_base + (uint32_t)(g * (kTmemCols / kGroups));
      ctx.mbar = &H->mbar[g];
      ctx.mma_phase = &H->mma_phase[g];
      ctx.aux = ctl->aux;
      ctx.flags = task->flags | ctl->plan;
      ctx.part = ctl->part;
      ctx.nparts = ctl->nparts;
      const uint32_t kind = ctl->kind;
      if (ctx.tid == 0) LAT_STAMP(6);
      if (!dense_f32_inline(kind, task, &ctx)) {
        OpFn fn;
        if (kind < kNumKinds) {
          fn = g_kind_fns[kind];
        } else {
          // native injected op, or its device program when this generation's
          // module does not carry the native code
          OpFn_ p = jit_fns ? jit_fns[kind - kJitKindBase] : nullptr;
          fn = p ? reinterpret_cast<OpFn>(p) : op_program;
        }
        code = fn(task, &ctx);
      }
      if (ctx.tid == 0) LAT_STAMP(7);
    }
    group_sync(&ctx);
    if (ctx.tid == 0) LAT_STAMP(8);
    if (ctx.tid == 0) {
      ctl->code = code;
      ctl->t_fenced = t_wake;
      ctl->t_end = ctl->trace_on ? globaltimer() : 0;
      mbar_arrive1(&H->done_bar[b]);
    }
  }
}

#ifndef GPUOS_WORKER_IMAGE  // the relocatable image for native ops carries only the worker
// ---------------------------------------------------------------------------
// Conventional path: the same bodies as standalone kernels, one launch per task.
// ---------------------------------------------------------------------------
template <int KIND>
__device__ __forceinline__ int body(const gpuos_task* t, const Ctx* c) {
  switch (KIND) {
    case GPUOS_OP_ADD: return op_add(t, c);
    case GPUOS_OP_MUL: return op_mul(t, c);
    case GPUOS_OP_RELU: return op_relu(t, c);
    case GPUOS_OP_GELU: return op_gelu(t, c);
    case GPUOS_OP_SOFTMAX: return op_softmax(t, c);
    case GPUOS_OP_LAYERNORM: return op_layernorm(t, c);
    case GPUOS_OP_REDUCE_SUM: return op_reduce_sum(t, c);
    case GPUOS_OP_REDUCE_MAX: return op_reduce_max(t, c);
    case GPUOS_OP_REDUCE_MIN: return op_reduce_min(t, c);
    case GPUOS_OP_MATMUL_SMALL: return op_matmul(t, c);
    case GPUOS_OP_VECMAT: return op_vecmat(t, c);
    case GPUOS_OP_SDPA: return op_sdpa(t, c);
    case GPUOS_OP_ROPE: return op_rope(t, c);
    case GPUOS_OP_KV_APPEND: return op_kv_append(t, c);
    case GPUOS_KIND_PROGRAM: return op_program(t, c);
    default: return GPUOS_OPERATOR_KILLED;
  }
}

template <int KIND>
// (256, 3): <= 80 registers, so a standalone kernel's warps fit the register
// quadrants an SM has left next to a resident worker CTA (9 warps x 96
// registers); with 128 registers the launch would wait for the generation
// to exit.
__global__ void __launch_bounds__(256, 3) gpuos_task_kernel(const gpuos_task task, uint64_t aux, uint32_t* counter) {
  extern __shared__ __align__(128) char tsmem[];
  char* smem = tsmem;
  gpuos_task* t = reinterpret_cast<gpuos_task*>(smem);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(&task);
  for (int i = threadIdx.x; i < (int)(sizeof(gpuos_task) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(t)[i] = src[i];
  uint32_t* plan_s = reinterpret_cast<uint32_t*>(smem + kTaskBytes);
  uint32_t* tmem_s = plan_s + 1;
  uint32_t* phase_s = plan_s + 2;
  uint64_t* mbar_s = reinterpret_cast<uint64_t*>(smem + kTaskBytes + 16);
  constexpr bool kTensor = KIND == GPUOS_OP_MATMUL_SMALL;
  if (kTensor) {
    if (threadIdx.x == 0) {
      mbar_init(mbar_s, 1);
      *phase_s = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) tmem_alloc(tmem_s, 128);
    tc_fence_before();
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const uint32_t plan = plan_task_warp(t, threadIdx.x);
    if (threadIdx.x == 0) *plan_s = plan;
  }
  __syncthreads();
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  Ctx ctx;
  ctx.tid = threadIdx.x;
  ctx.nthreads = blockDim.x;
  ctx.part = blockIdx.x;
  ctx.nparts = gridDim.x;
  ctx.bar_id = 1;
  ctx.smem = smem + kTaskBytes + kCtlBytes;
  ctx.smem_bytes = (int)dyn - (int)(kTaskBytes + kCtlBytes);
  ctx.aux = aux;
  ctx.flags = t->flags | *plan_s;
  if (kTensor) tc_fence_after();
  ctx.tmem = kTensor ? *tmem_s : kNoTmem;
  ctx.mbar = mbar_s;
  ctx.mma_phase = phase_s;
  const int code = body<KIND>(t, &ctx);
  if (kTensor) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc(*tmem_s, 128);
  }
  __syncthreads();
  if (threadIdx.x == 0 && t->done_cell) {
    bool last = true;
    if (gridDim.x > 1) {
      __threadfence();
      last = atomicAdd(counter, 1u) == gridDim.x - 1;
      if (last) *counter = 0;
    }
    if (last) {
      fence_acq_rel_sys();
      const uint64_t word = ((uint64_t)(code == GPUOS_OK ? 1 : 2)) | ((uint64_t)(code & 0xff) << 8) | (t->seq << 16);
      st_relaxed_sys((uint64_t*)t->done_cell, word);
    }
  }
}

// Host <-> device clock ping-pong: round r waits for the host's flag to reach
// r + 1 (mapped memory) and answers with %globaltimer; the host brackets each
// round with its steady clock, so the offset error is half the round trip.
__global__ void gpuos_clock_probe(const uint32_t* flag, uint64_t* out, int rounds) {
  if (!flag) {  // one-shot stamp (under a profiler, which serialises launches)
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(globaltimer()) : "memory");
    return;
  }
  for (int r = 0; r < rounds; ++r) {
    uint32_t f;
    do {
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
    } while (f < (uint32_t)(r + 1));
    const uint64_t t = globaltimer();
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out + r), "l"(t) : "memory");
  }
}

// Lean per-op baseline: what a conventional CUDA program launches for one
// dense f32 add -- four small parameters, no descriptor, no dynamic shared
// memory, a grid sized to the op (bench.py's second per-op-launch arm).
__global__ void __launch_bounds__(256) gpuos_lean_add_kernel(float* out, const float* a, const float* b, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nv = n / 4;
  if (i < nv) {
    const float4 x = reinterpret_cast<const float4*>(a)[i], y = reinterpret_cast<const float4*>(b)[i];
    reinterpret_cast<float4*>(out)[i] = make_float4(__fadd_rn(x.x, y.x), __fadd_rn(x.y, y.y), __fadd_rn(x.z, y.z),
                                                    __fadd_rn(x.w, y.w));
  }
  for (int e = nv * 4 + i; e < n && i < 4; e += 4) out[e] = __fadd_rn(a[e], b[e]);
}

__global__ void gpuos_gen_init(DevState* S, uint64_t claim, uint64_t hint, uint64_t stop_pos) {
  S->claim = claim;
  S->hint = hint;
  S->stop_pos = stop_pos;
}

typedef void (*TaskKernel)(const gpuos_task, uint64_t, uint32_t*);

static TaskKernel task_kernel_for(uint32_t kind) {
  if (kind >= kJitKindBase && kind < kJitKindBase + kJitSlots) kind = GPUOS_KIND_PROGRAM;
  switch (kind) {
    case GPUOS_OP_ADD: return gpuos_task_kernel<GPUOS_OP_ADD>;
    case GPUOS_OP_MUL: return gpuos_task_kernel<GPUOS_OP_MUL>;
    case GPUOS_OP_RELU: return gpuos_task_kernel<GPUOS_OP_RELU>;
    case GPUOS_OP_GELU: return gpuos_task_kernel<GPUOS_OP_GELU>;
    case GPUOS_OP_SOFTMAX: return gpuos_task_kernel<GPUOS_OP_SOFTMAX>;
    case GPUOS_OP_LAYERNORM: return gpuos_task_kernel<GPUOS_OP_LAYERNORM>;
    case GPUOS_OP_REDUCE_SUM: return gpuos_task_kernel<GPUOS_OP_REDUCE_SUM>;
    case GPUOS_OP_REDUCE_MAX: return gpuos_task_kernel<GPUOS_OP_REDUCE_MAX>;
    case GPUOS_OP_REDUCE_MIN: return gpuos_task_kernel<GPUOS_OP_REDUCE_MIN>;
    case GPUOS_OP_MATMUL_SMALL: return gpuos_task_kernel<GPUOS_OP_MATMUL_SMALL>;
    case GPUOS_OP_VECMAT: return gpuos_task_kernel<GPUOS_OP_VECMAT>;
    case GPUOS_OP_SDPA: return gpuos_task_kernel<GPUOS_OP_SDPA>;
    case GPUOS_OP_ROPE: return gpuos_task_kernel<GPUOS_OP_ROPE>;
    case GPUOS_OP_KV_APPEND: return gpuos_task_kernel<GPUOS_OP_KV_APPEND>;
    case GPUOS_KIND_PROGRAM: return gpuos_task_kernel<GPUOS_KIND_PROGRAM>;
    default: return gpuos_task_kernel<GPUOS_KIND_KILLED>;
  }
}

uint32_t worker_smem_bytes() { return kHeaderBytes + kScratchBytes; }
// standalone task kernels: descriptor + control block + 64 KB scratch
uint32_t task_smem_bytes() { return kTaskBytes + kCtlBytes + 64 * 1024; }
uint32_t worker_threads() { return kWorkerThreads; }
int smem_carveout() {
  const char* e = std::getenv("GPUOS_CARVEOUT");
  return e ? std::atoi(e) : (int)cudaSharedmemCarveoutMaxShared;
}

// Lazy module loading blocks while the persistent kernel is resident
// (measured: profiles/r01_probe2_lazy.log), so every kernel is loaded and
// configured before the first worker launch.
void load_all_kernels(int* worker_regs, size_t* worker_local) {
  const uint32_t smem = worker_smem_bytes();
  cudaFuncSetAttribute(gpuos_worker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // every kernel asks for the largest shared carveout, so an SM configured by
  // the resident worker also has room for a standalone task kernel
  cudaFuncSetAttribute(gpuos_worker_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, smem_carveout());
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gpuos_worker_kernel);
  if (worker_regs) *worker_regs = fa.numRegs;
  if (worker_local) *worker_local = fa.localSizeBytes;
  const uint32_t kinds[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, GPUOS_KIND_PROGRAM, GPUOS_KIND_KILLED};
  for (uint32_t k : kinds) {
    TaskKernel f = task_kernel_for(k);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, task_smem_bytes());
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, smem_carveout());
    cudaFuncGetAttributes(&fa, f);
  }
  cudaFuncGetAttributes(&fa, gpuos_clock_probe);
  cudaFuncGetAttributes(&fa, gpuos_gen_init);
  cudaFuncGetAttributes(&fa, gpuos_lean_add_kernel);
}

cudaError_t worker_occupancy(int* per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, gpuos_worker_kernel, kWorkerThreads, worker_smem_bytes());
}

cudaError_t launch_worker(DevState* s, uint32_t workers, uint32_t threads, uint32_t smem, cudaStream_t st) {
  void* args[] = {&s};
  return cudaLaunchKernel((const void*)gpuos_worker_kernel, dim3(workers), dim3(threads), args, smem, st);
}

cudaError_t launch_task(const gpuos_task* t, uint32_t kind, uint64_t aux, uint32_t nparts, uint32_t* counter,
                        cudaStream_t st) {
  TaskKernel f = task_kernel_for(kind);
  void* args[] = {(void*)t, &aux, &counter};
  return cudaLaunchKernel((const void*)f, dim3(nparts), dim3(256), args, task_smem_bytes(), st);
}

cudaError_t launch_clock_probe(const uint32_t* flag, uint64_t* out, int rounds, cudaStream_t st) {
  gpuos_clock_probe<<<1, 1, 0, st>>>(flag, out, rounds);
  return cudaGetLastError();
}

cudaError_t launch_lean_add(float* out, const float* a, const float* b, int n, cudaStream_t st) {
  const int nv = (n + 3) / 4;
  gpuos_lean_add_kernel<<<(nv + 255) / 256, 256, 0, st>>>(out, a, b, n);
  return cudaGetLastError();
}

cudaError_t launch_gen_init(DevState* s, uint64_t claim, uint64_t hint, uint64_t stop_pos, cudaStream_t st) {
  gpuos_gen_init<<<1, 1, 0, st>>>(s, claim, hint, stop_pos);
  return cudaGetLastError();
}

#endif  // GPUOS_WORKER_IMAGE

}  // namespace gdev
