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
  uint32_t kind;
  int32_t code;
  uint32_t exit;
  uint32_t pad;
};

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

// Warp 0: claim one ticket, wait for its publication, copy it to shared
// memory, free the slot, and resolve the op through the versioned table.
__device__ __forceinline__ void claim_and_fetch(DevState* S, uint32_t w, gpuos_task* task, SharedCtl* ctl,
                                                uint64_t& my_epoch, uint64_t& claimed, int lane) {
  uint64_t pos = 0;
  if (lane == 0) pos = atomicAdd((unsigned long long*)&S->claim, 1ull);
  pos = shfl64(pos, 0);
  const char* slot = (const char*)(S->ring + (pos & S->mask));
  uint32_t spins = 0, expn = 0;
  bool quiesced = false;
  uint4 v = make_uint4(0, 0, 0, 0);
  for (;;) {
    const uint64_t sp = ld_relaxed_gpu(&S->stop_pos);
    if (pos > sp) {
      if (lane == 0) {
        quiesce(S, w);
        ctl->exit = 1;
      }
      return;
    }
    const uint64_t h = ld_relaxed_gpu(&S->hint);
    const bool near = pos < h + 2;
    if (near || (spins & 7) == 0) {
      if (lane < 24) v = ld_volatile_v4(slot + 16 * lane);
      uint64_t tail = 0;
      if (lane == 24) tail = ld_relaxed_sys(S->host_tail);
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
    if (!quiesced && spins >= S->spin_iterations) {
      // Parked workers must not pin a table version (executor.hpp:160-161).
      if (lane == 0) {
        quiesce(S, w);
        atomicAdd((unsigned long long*)&S->stalls, 1ull);
      }
      quiesced = true;
      my_epoch = kQuiescent;
    }
    if (!near) {
      __nanosleep(64u << expn);
      if (expn < S->backoff_max_exp) ++expn;
    }
  }
  // fetched: stage the descriptor in shared memory
  if (lane < 24) reinterpret_cast<uint4*>(task)[lane] = v;
  __syncwarp();
  if (lane == 0) {
    // free the slot for the producer's next lap, then acquire: the host
    // published the descriptor after the inputs were written.
    st_relaxed_sys((uint64_t*)(S->ring + (pos & S->mask)), pos + S->cap);
    fence_acq_rel_sys();
    ++claimed;
    st_relaxed_sys(&S->host_claimed[w], claimed);
    ctl->pos = pos;
    ctl->exit = 0;
    ctl->t_deq = globaltimer();
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
    }
  }
  __syncwarp();
}

extern "C" __global__ void __launch_bounds__(256, 2) gpuos_worker_kernel(DevState* S) {
  extern __shared__ __align__(128) char smem[];
  gpuos_task* task = reinterpret_cast<gpuos_task*>(smem);
  SharedCtl* ctl = reinterpret_cast<SharedCtl*>(smem + kTaskBytes);
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
  ctx.smem = smem + kTaskBytes + kCtlBytes;
  ctx.smem_bytes = (int)dyn - (int)(kTaskBytes + kCtlBytes);
  ctx.aux = 0;
  ctx.flags = 0;
  uint64_t my_epoch = kQuiescent, claimed = 0, done = 0, executed = 0;
  if (tid == 0) {
    // continue the host-visible counts across kernel generations
    claimed = ld_relaxed_sys(&S->host_claimed[w]);
    done = ld_relaxed_sys(&S->host_done[w]);
  }
  for (;;) {
    if (warp == 0) claim_and_fetch(S, w, task, ctl, my_epoch, claimed, lane);
    __syncthreads();
    if (ctl->exit) return;
    int code = ctl->code;
    if (code == GPUOS_OK) {
      ctx.aux = ctl->aux;
      ctx.flags = task->flags;
      const OpFn fn = g_kind_fns[ctl->kind];
      code = fn(task, &ctx);
    }
    __syncthreads();
    if (tid == 0) {
      const uint64_t t_end = globaltimer();
      // completion (runtime.hpp:628-639): outputs of every thread are ordered
      // before the system-scope release through the barrier above.
      fence_acq_rel_sys();
      if (task->done_cell) {
        const uint64_t word = ((uint64_t)(code == GPUOS_OK ? 1 : 2)) | ((uint64_t)(code & 0xff) << 8) |
                              (task->seq << 16);
        st_relaxed_sys((uint64_t*)task->done_cell, word);
      }
      ++done;
      st_relaxed_sys(&S->host_done[w], done);
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
        __threadfence();
        r->stamp = ticket * 2 + 2;
      }
      ++executed;
      const uint64_t ye = ld_relaxed_gpu(&S->yield_every);
      if (ye > 0 && executed % ye == 0) __nanosleep(1000);  // yield_every (executor.hpp:190-193)
    }
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

uint32_t worker_smem_bytes() { return kTaskBytes + kCtlBytes + kScratchBytes; }

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
