// The persistent sm_100a worker kernel (reference Executor, executor.hpp:45-278,
// re-designed as one resident CTA per worker), the module jump table, and the
// standalone per-task kernels of the conventional path (execute_inline,
// runtime.hpp:567-619 == baseline (a): one cudaLaunchKernel per task).
//
// Claim protocol (queue.hpp:179-261 restated for PCIe):
//   * warp 0, lane 0 takes a ticket `pos` with atomicAdd on the HBM claim
//     cursor; tickets are FIFO, so the shutdown sentinel drains all earlier
//     work (executor.hpp:178-184).
//   * the warp polls slot pos in mapped pinned memory with one 384-byte
//     warp-wide volatile load (24 lanes x 16 B) plus the producer tail
//     (lane 24); publication = slot word 0 == pos+1, torn reads are caught by
//     a warp-reduced checksum (queue.hpp:249-251).  Only tickets within two
//     of the highest tail seen on the device poll PCIe continuously; the rest
//     back off on an HBM hint, so idle PCIe traffic stays small.
//   * lane 0 frees the slot (word 0 = pos + capacity, queue.hpp:248), mirrors
//     its claimed count to host memory, snapshots the table version with the
//     publish-then-revalidate epoch protocol (executor.hpp:133-141), and looks
//     the op up in the bank of that version with the generation canary
//     (executor.hpp:197-212).
//   * all warps run the task body; thread 0 posts the completion word with a
//     system-scope release and the per-worker processed count.
#include "dev_common.cuh"
#include "dev_state.h"
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
  uint64_t t_fenced;
  uint32_t kind;
  int32_t code;
  uint32_t exit;
  uint32_t pad;
};

constexpr uint32_t kCtlStride = 112;
static_assert(sizeof(SharedCtl) <= kCtlStride, "SharedCtl must fit its stride");

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// Publish-then-revalidate (executor.hpp:133-141): the epoch slot holds the
// version dispatched under before any bank is read.
__device__ __forceinline__ uint64_t stable_snapshot(DevState* S, uint32_t w, uint64_t v) {
  for (;;) {
    st_relaxed_gpu(&S->dev_epoch[w], v);
    st_relaxed_sys(&S->host_epoch[w], v);
    fence_sc_sys();
    const uint64_t now = ld_acquire_gpu(&S->version);
    if (now == v) return v;
    v = now;
  }
}

__device__ __forceinline__ void quiesce(DevState* S, uint32_t w) {
  st_relaxed_gpu(&S->dev_epoch[w], kQuiescent);
  st_relaxed_sys(&S->host_epoch[w], kQuiescent);
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

// Host-visible per-worker counts are written lazily by warp 0 lane 0 (the
// single writer, so posted writes stay monotone): every 16 claims and on every
// idle poll where they changed, and once more at exit.
struct Mirror {
  uint64_t claimed = 0, flushed_claimed = 0, flushed_done = 0;
};
__device__ __forceinline__ void flush_mirror(DevState* S, uint32_t w, Mirror& m, uint64_t done) {
  if (m.claimed != m.flushed_claimed) {
    st_relaxed_sys(&S->host_claimed[w], m.claimed);  // claimed before done: head >= processed
    m.flushed_claimed = m.claimed;
  }
  if (done != m.flushed_done) {
    st_relaxed_sys(&S->host_done[w], done);
    m.flushed_done = done;
  }
}

// Warp 0: claim one ticket, wait for its publication, copy it to shared
// memory, free the slot, and resolve the op through the versioned table.
//
// PCIe discipline (measured, profiles/r01_phases_*.log): every host-memory
// access costs a round trip through the VM's PCIe path and a fence that
// follows a sysmem store waits for it, so this path issues one slot read, one
// slot-free store, the tail read only when the ticket is past the hint, and no
// fence.  Task inputs need no acquire fence because the worker module is
// compiled with -dlcm=cg: global loads bypass the (non-coherent) L1.
//
// Epochs: an idle worker does not park; every 16 polls it re-reads the table
// version and republishes its epoch when the version moved, so an install's
// epoch wait (optable.hpp:591-600) completes within a few polls while the
// common claim path pays no system-scope fence when the version is unchanged.
__device__ __forceinline__ void claim_and_fetch(DevState* S, uint32_t w, gpuos_task* task, SharedCtl* ctl,
                                                uint64_t& my_epoch, Mirror& mir, const volatile uint64_t* done,
                                                int lane) {
  uint64_t pos = 0;
  if (lane == 0) {
    while (*(volatile uint32_t*)&S->hold) __nanosleep(2000);
    pos = atomicAdd((unsigned long long*)&S->claim, 1ull);
  }
  pos = shfl64(pos, 0);
  const uint64_t t_ticket = globaltimer();
  const char* slot = (const char*)(S->ring + (pos & S->mask));
  uint32_t spins = 0, expn = 0;
  uint4 v = make_uint4(0, 0, 0, 0);
  for (;;) {
    const uint64_t sp = ld_relaxed_gpu(&S->stop_pos);
    if (pos > sp) {
      if (lane == 0) {
        quiesce(S, w);
        my_epoch = kQuiescent;
        ctl->exit = 1;
      }
      return;
    }
    // Only tickets within two of the highest tail seen on the device read
    // PCIe; the rest watch the HBM hint.  Progress: the ticket equal to the
    // hint is always near, and its poll carries the producer tail (lane 24),
    // so every publication eventually advances the hint.
    const uint64_t h = ld_relaxed_gpu(&S->hint);
    const bool near = pos < h + 2;
    if (near) {
      if (lane < 24) v = ld_volatile_v4(slot + 16 * lane);
      uint64_t tail = 0;
      if (lane == 24 && pos >= h) tail = ld_relaxed_sys(S->host_tail);
      const uint64_t pub = ((uint64_t)__shfl_sync(0xffffffffu, v.y, 0) << 32) | __shfl_sync(0xffffffffu, v.x, 0);
      tail = shfl64(tail, 24);
      if (lane == 0 && tail > h) atomicMax((unsigned long long*)&S->hint, (unsigned long long)tail);
      if (pub == pos + 1) {
        const uint64_t w0 = ((uint64_t)v.y << 32) | v.x, w1 = ((uint64_t)v.w << 32) | v.z;
        uint64_t part = 0;
        if (lane < 24) {
          part = slot_mix(w0, 2 * lane);
          if (lane != 3) part += slot_mix(w1, 2 * lane + 1);  // word 7 is the checksum
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        const uint64_t chk = shfl64(w1, 3);
        if (part == chk) break;
        if (lane == 0) atomicAdd((unsigned long long*)&S->torn_reads, 1ull);
        continue;  // torn: re-read immediately
      }
    }
    ++spins;
    if (lane == 0) {
      flush_mirror(S, w, mir, *done);  // idle: make counts visible to wait_all / peek
      if ((spins & 15) == 0) {
        const uint64_t ver = ld_acquire_gpu(&S->version);
        if (ver != my_epoch) my_epoch = stable_snapshot(S, w, ver);
        if (spins == S->spin_iterations) atomicAdd((unsigned long long*)&S->stalls, 1ull);
      }
    }
    if (!near) {
      __nanosleep(64u << expn);
      if (expn < S->backoff_max_exp) ++expn;
    }
  }
  const uint64_t t_seen = globaltimer();
  // fetched: stage the descriptor in shared memory
  if (lane < 24) reinterpret_cast<uint4*>(task)[lane] = v;
  __syncwarp();
  if (lane == 0) {
    // free the slot for the producer's next lap (queue.hpp:248)
    st_relaxed_sys((uint64_t*)(S->ring + (pos & S->mask)), pos + S->cap);
    ++mir.claimed;
    if ((mir.claimed & 15) == 0) flush_mirror(S, w, mir, *done);
    ctl->t_fenced = globaltimer();
    ctl->pos = pos;
    ctl->exit = 0;
    ctl->t_ticket = t_ticket;
    ctl->t_seen = t_seen;
    if (task->flags & GPUOS_FLAG_SHUTDOWN) {
      atomicMin((unsigned long long*)&S->stop_pos, (unsigned long long)pos);
      quiesce(S, w);
      my_epoch = kQuiescent;
      ctl->exit = 1;
    } else {
      uint64_t ver = ld_acquire_gpu(&S->version);
      if (ver != my_epoch) ver = stable_snapshot(S, w, ver);
      my_epoch = ver;
      const uint32_t op = task->op_id;
      int code = GPUOS_OK;
      TableEntry e;
      e.kind = 0;
      e.aux = 0;
      for (int retry = 0;; ++retry) {
        if (op >= S->table_slots) {
          code = GPUOS_OUT_OF_RANGE;
          break;
        }
        e = load_entry(&S->bank[ver & 1][op]);
        const uint64_t gen = ld_relaxed_gpu(&S->bank_gen[ver & 1]);
        code = e.status == 1 ? GPUOS_OK : (e.status == 2 ? GPUOS_OPERATOR_KILLED : GPUOS_NOT_INSTALLED);
        // canary: an entry must carry the generation of its version's bank
        if (code == GPUOS_OK && gen != ver && retry < 4) {
          atomicAdd((unsigned long long*)&S->canary_hits, 1ull);
          ver = stable_snapshot(S, w, ld_acquire_gpu(&S->version));
          my_epoch = ver;
          continue;
        }
        break;
      }
      ctl->version = ver;
      ctl->code = code;
      ctl->kind = e.kind < kNumKinds ? e.kind : (uint32_t)GPUOS_KIND_KILLED;
      ctl->aux = e.aux;
      ctl->t_deq = globaltimer();
    }
  }
  __syncwarp();
}

// Completion (runtime.hpp:628-639) by lane 0 of one of warps 1..7, rotating
// per task, while warp 0 already claims the next task into the other buffer.
// Every thread's outputs are ordered before it by the barrier; the gpu-scope
// release puts them in L2 (where the host's copy engine reads) before the
// word is posted.  Rotating the completer means the fence never waits on a
// sysmem store issued by the same warp just before.
__device__ __forceinline__ void complete_task(DevState* S, uint32_t w, const gpuos_task* task, const SharedCtl* ctl,
                                              int code, volatile uint64_t* done, uint64_t& executed) {
  const uint64_t t_end = globaltimer();
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (task->done_cell) {
    const uint64_t word = ((uint64_t)(code == GPUOS_OK ? 1 : 2)) | ((uint64_t)(code & 0xff) << 8) | (task->seq << 16);
    st_relaxed_sys((uint64_t*)task->done_cell, word);
  }
  *done = *done + 1;
  atomicAdd((unsigned long long*)&S->processed, 1ull);
  if (code != GPUOS_OK) atomicAdd((unsigned long long*)&S->failed, 1ull);
  atomicAdd((unsigned long long*)&S->per_op[task->op_id < 256 ? task->op_id : 255], 1ull);
  if (S->trace_on) {
    const uint64_t ticket = atomicAdd((unsigned long long*)&S->trace_head, 1ull);
    TraceRec* r = &S->trace[ticket % S->trace_cap];
    r->stamp = ticket * 2 + 1;
    r->seq = task->seq;
    r->op_id = task->op_id;
    r->worker = w;
    r->enqueue_ns = task->enqueue_ns;
    r->dequeue_gt = ctl->t_deq;
    r->exec_ns = t_end > ctl->t_deq ? t_end - ctl->t_deq : 1;
    r->version = ctl->version;
    r->t_ticket = ctl->t_ticket;
    r->t_seen = ctl->t_seen;
    r->t_done = globaltimer();
    r->pad = ctl->t_fenced;
    __threadfence();
    r->stamp = ticket * 2 + 2;
  }
  ++executed;
  const uint64_t ye = ld_relaxed_gpu(&S->yield_every);
  if (ye > 0 && executed % ye == 0) __nanosleep(1000);  // yield_every (executor.hpp:190-193)
}

extern "C" __global__ void __launch_bounds__(256, 2) gpuos_worker_kernel(DevState* S) {
  extern __shared__ __align__(128) char smem[];
  // two task buffers: warp 0 fetches task k+1 while task k is being completed
  gpuos_task* tasks[2] = {reinterpret_cast<gpuos_task*>(smem), reinterpret_cast<gpuos_task*>(smem + kTaskBytes)};
  // header layout: task[0] | task[1] | ctl[0] | ctl[1] | done counter
  static_assert(2 * kTaskBytes + 2 * kCtlStride + 8 <= kHeaderBytes, "worker header overflows");
  SharedCtl* ctls[2] = {reinterpret_cast<SharedCtl*>(smem + 2 * kTaskBytes),
                        reinterpret_cast<SharedCtl*>(smem + 2 * kTaskBytes + kCtlStride)};
  volatile uint64_t* done = reinterpret_cast<volatile uint64_t*>(smem + 2 * kTaskBytes + 2 * kCtlStride);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t w = blockIdx.x;
  uint32_t dyn;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
  Ctx ctx;
  ctx.tid = tid;
  ctx.nthreads = blockDim.x;
  ctx.part = 0;
  ctx.nparts = 1;
  ctx.bar_id = 1;
  ctx.smem = smem + kHeaderBytes;
  ctx.smem_bytes = (int)dyn - (int)kHeaderBytes;
  ctx.aux = 0;
  ctx.flags = 0;
  uint64_t my_epoch = kQuiescent, executed = 0;
  Mirror mir;
  if (tid == 0) {
    // continue the host-visible counts across kernel generations
    mir.claimed = mir.flushed_claimed = ld_relaxed_sys(&S->host_claimed[w]);
    mir.flushed_done = ld_relaxed_sys(&S->host_done[w]);
    *done = mir.flushed_done;
  }
  __syncthreads();
  const int nwarps = blockDim.x >> 5;
  uint32_t k = 0;
  for (;; ++k) {
    gpuos_task* task = tasks[k & 1];
    SharedCtl* ctl = ctls[k & 1];
    if (warp == 0) claim_and_fetch(S, w, task, ctl, my_epoch, mir, done, lane);
    __syncthreads();
    if (ctl->exit) {
      if (tid == 0) flush_mirror(S, w, mir, *done);  // final counts for wait_all and the next generation
      return;
    }
    int code = ctl->code;
    if (code == GPUOS_OK) {
      ctx.aux = ctl->aux;
      ctx.flags = task->flags;
      const OpFn fn = g_kind_fns[ctl->kind];
      code = fn(task, &ctx);
    }
    __syncthreads();
    if (lane == 0 && warp == 1 + (int)(k % (uint32_t)(nwarps - 1))) complete_task(S, w, task, ctl, code, done, executed);
  }
}

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
__global__ void __launch_bounds__(256, 2) gpuos_task_kernel(const gpuos_task task, uint64_t aux, uint32_t* counter) {
  extern __shared__ __align__(128) char tsmem[];
  char* smem = tsmem;
  gpuos_task* t = reinterpret_cast<gpuos_task*>(smem);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(&task);
  for (int i = threadIdx.x; i < (int)(sizeof(gpuos_task) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(t)[i] = src[i];
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
  ctx.flags = t->flags;
  const int code = body<KIND>(t, &ctx);
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

__global__ void gpuos_clock_probe(uint64_t* out) { out[0] = globaltimer(); }

typedef void (*TaskKernel)(const gpuos_task, uint64_t, uint32_t*);

static TaskKernel task_kernel_for(uint32_t kind) {
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

// Lazy module loading blocks while the persistent kernel is resident
// (measured: profiles/r01_probe2_lazy.log), so every kernel is loaded and
// configured before the first worker launch.
void load_all_kernels(int* worker_regs, size_t* worker_local) {
  const uint32_t smem = worker_smem_bytes();
  cudaFuncSetAttribute(gpuos_worker_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, gpuos_worker_kernel);
  if (worker_regs) *worker_regs = fa.numRegs;
  if (worker_local) *worker_local = fa.localSizeBytes;
  const uint32_t kinds[] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, GPUOS_KIND_PROGRAM, GPUOS_KIND_KILLED};
  for (uint32_t k : kinds) {
    TaskKernel f = task_kernel_for(k);
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncGetAttributes(&fa, f);
  }
  cudaFuncGetAttributes(&fa, gpuos_clock_probe);
}

cudaError_t launch_worker(DevState* s, uint32_t workers, uint32_t threads, uint32_t smem, cudaStream_t st) {
  void* args[] = {&s};
  return cudaLaunchKernel((const void*)gpuos_worker_kernel, dim3(workers), dim3(threads), args, smem, st);
}

cudaError_t launch_task(const gpuos_task* t, uint32_t kind, uint64_t aux, uint32_t nparts, uint32_t* counter,
                        cudaStream_t st) {
  TaskKernel f = task_kernel_for(kind);
  void* args[] = {(void*)t, &aux, &counter};
  return cudaLaunchKernel((const void*)f, dim3(nparts), dim3(256), args, worker_smem_bytes(), st);
}

cudaError_t launch_clock_probe(uint64_t* out, cudaStream_t st) {
  gpuos_clock_probe<<<1, 1, 0, st>>>(out);
  return cudaGetLastError();
}

}  // namespace gdev
