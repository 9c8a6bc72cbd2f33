/*
 * gpuos_cuda.h — the C-ABI drop-in boundary of the B200-native GPUOS runtime.
 *
 * Everything CUDA (device memory, the persistent worker kernel, the task
 * ring in mapped pinned memory, the dual-bank device operator table, the
 * injected-operator programs, the per-op cudaLaunchKernel baseline and
 * NVRTC) lives behind these extern "C" entry points in libgpuos_cuda.so.
 * Signatures use plain integers, pointers and sizes only: no CUDA, torch or
 * C++ types.  Every function returns an int ErrorCode (0 = Ok) and never
 * throws.
 *
 * The C++ host runtime (paper_2604_17861_b200/include/gpuos/runtime.hpp)
 * keeps the reference's public API (reference: proj/include/gpuos/
 * runtime.hpp:205-450) and calls only this header.  Each entry point cites
 * the reference interface it replaces.
 */
#ifndef GPUOS_CUDA_H_
#define GPUOS_CUDA_H_

#ifdef __CUDACC_RTC__  /* NVRTC (natively compiled injected ops): no libc headers */
#include <cuda/std/cstddef>
#include <cuda/std/cstdint>
typedef cuda::std::size_t size_t;
typedef cuda::std::int8_t int8_t;
typedef cuda::std::int16_t int16_t;
typedef cuda::std::int32_t int32_t;
typedef cuda::std::int64_t int64_t;
typedef cuda::std::uint8_t uint8_t;
typedef cuda::std::uint16_t uint16_t;
typedef cuda::std::uint32_t uint32_t;
typedef cuda::std::uint64_t uint64_t;
typedef cuda::std::uintptr_t uintptr_t;
#else
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define GPUOS_ABI_VERSION 1

/* ---- error codes: identical integer values to gpuos::ErrorCode
 *      (reference errors.hpp:9-41) so codes cross the ABI unchanged ---- */
enum gpuos_error {
  GPUOS_OK = 0,
  GPUOS_INCOMPATIBLE_SHAPES = 1,
  GPUOS_OUT_OF_BOUNDS = 2,
  GPUOS_INVALID_BUFFER = 3,
  GPUOS_ZERO_CAPACITY = 4,
  GPUOS_QUEUE_FULL = 5,
  GPUOS_ZERO_SLOTS = 6,
  GPUOS_OUT_OF_RANGE = 7,
  GPUOS_NOT_INSTALLED = 8,
  GPUOS_OPERATOR_KILLED = 9,
  GPUOS_TABLE_FULL = 10,
  GPUOS_SYNTAX_ERROR = 11,
  GPUOS_UNKNOWN_IDENTIFIER = 12,
  GPUOS_ARITY_ERROR = 13,
  GPUOS_VERIFY_ERROR = 14,
  GPUOS_EMPTY_AXIS = 15,
  GPUOS_DTYPE_MISMATCH = 16,
  GPUOS_SHAPE_MISMATCH = 17,
  GPUOS_TOO_LARGE = 18,
  GPUOS_ODD_DIM = 19,
  GPUOS_CACHE_FULL = 20,
  GPUOS_ALREADY_STARTED = 21,
  GPUOS_RUNTIME_STOPPED = 22,
  GPUOS_IO_ERROR = 23,
  GPUOS_INTERNAL = 24
};

/* ---- dtypes: F32/F64/I32 keep the reference values (tensor.hpp:24);
 *      F16/BF16 are new in this build ---- */
enum gpuos_dtype { GPUOS_F32 = 0, GPUOS_F64 = 1, GPUOS_I32 = 2, GPUOS_F16 = 3, GPUOS_BF16 = 4 };

/* ---- builtin operator kinds = fixed op ids (reference ops.hpp:31-48) ---- */
enum gpuos_op_kind {
  GPUOS_OP_ADD = 0,
  GPUOS_OP_MUL = 1,
  GPUOS_OP_RELU = 2,
  GPUOS_OP_GELU = 3,
  GPUOS_OP_SOFTMAX = 4,
  GPUOS_OP_LAYERNORM = 5,
  GPUOS_OP_REDUCE_SUM = 6,
  GPUOS_OP_REDUCE_MAX = 7,
  GPUOS_OP_REDUCE_MIN = 8,
  GPUOS_OP_MATMUL_SMALL = 9,
  GPUOS_OP_VECMAT = 10,
  GPUOS_OP_SDPA = 11,
  GPUOS_OP_ROPE = 12,
  GPUOS_OP_KV_APPEND = 13,
  GPUOS_NUM_BUILTINS = 14,
  /* device-side bodies that are not reference op ids */
  GPUOS_KIND_PROGRAM = 64, /* elementwise stack-machine program (injected ops) */
  GPUOS_KIND_KILLED = 65   /* fail-fast stub installed by kill (optable.hpp:135-142) */
};

#define GPUOS_MAX_INPUTS 4      /* queue.hpp:27 */
#define GPUOS_MAX_SCALARS 8     /* queue.hpp:28 */
#define GPUOS_MAX_RANK 4        /* queue.hpp:29 (inline rank) */
#define GPUOS_SLOT_BYTES 384    /* one ring slot = one gpuos_task */
#define GPUOS_FIRST_INJECTED_ID 32u   /* ops.hpp:49 */
#define GPUOS_COMPOSITE_OP_ID 31u     /* runtime.hpp:41 */
#define GPUOS_SMALL_MATMUL_MAX_DIM 256 /* ops.hpp:53 */

/* task flags (queue.hpp:22-25) */
#define GPUOS_FLAG_FUSED_COMPOSITE 0x1u
#define GPUOS_FLAG_SHUTDOWN 0x2u
#define GPUOS_FLAG_UNCAPPED 0x4u /* matmul/vecmat without the 256 cap (inline path, runtime.hpp:589-594) */
/* Device-side ordering (extension; the reference has no inter-task ordering,
 * runtime.hpp:7-9): the task is handed to an executor only after the device's
 * processed count (gpuos_stats.processed) reaches the target carried in
 * gpuos_task.enqueue_ns (gpuos_dense_task.wait_target), i.e. after every task
 * committed before the fence that set the target has completed.  Such tasks
 * carry no enqueue stamp in the trace. */
#define GPUOS_FLAG_AFTER 0x8u
/* A GPUOS_FLAG_FUSED_COMPOSITE task (op id GPUOS_COMPOSITE_OP_ID) carries, in
 * scalars[0], the bits of the device address of its fused program (see
 * gpuos_program_upload) and, in scalars[1], the bits of the device address of
 * a completion record in mapped pinned memory: { n, cell_0, seq_0, ...,
 * cell_{n-1}, seq_{n-1} } for the chain's earlier steps, completed together
 * with the task's own done_cell (runtime.hpp:764-908). */
#define GPUOS_MAX_FUSED 15

/* Per-view bind status, resolved on the host at submit and surfaced by the
 * task body at the point where the reference constructs BoundView
 * (tensor.hpp:337-343), so error codes and accounting match. */
enum gpuos_view_status {
  GPUOS_VIEW_OK = 0,
  GPUOS_VIEW_UNKNOWN_BUFFER = 1,  /* -> InvalidBuffer */
  GPUOS_VIEW_DTYPE_VS_BUFFER = 2, /* -> DTypeMismatch */
  GPUOS_VIEW_OUT_OF_BOUNDS = 3    /* -> OutOfBounds (UB in the reference; checked here) */
};

/* A resolved strided view: 48 bytes.  `addr` is the device address of the
 * view's element 0 (buffer base + offset * width), so negative strides and
 * offsets need no base on the device.  Extents/strides are in elements and
 * fit int32 (queue.hpp:108-117 inline rule). */
typedef struct gpuos_view {
  uint64_t addr;
  int32_t extents[GPUOS_MAX_RANK];
  int32_t strides[GPUOS_MAX_RANK];
  uint8_t dtype;
  uint8_t rank;
  uint8_t status;
  uint8_t reserved;
  uint32_t buffer_lo; /* low bits of the BufferId, diagnostics only */
} gpuos_view;

/* One task descriptor == one ring slot (384 bytes, three 128-byte lines).
 * Replaces TaskDescriptor / PackedDescriptor (queue.hpp:38-90). */
typedef struct gpuos_task {
  uint64_t pub;        /* slot publication word; written by gpuos_ring_publish */
  uint64_t seq;        /* task sequence number (handle id) */
  uint32_t op_id;
  uint16_t flags;
  uint8_t n_inputs;
  uint8_t n_scalars;
  uint64_t size;       /* output element count */
  uint64_t done_cell;  /* device-visible address of an 8-byte completion cell, 0 = none */
  uint64_t enqueue_ns; /* host steady_clock at commit */
  uint64_t aux;        /* reserved */
  uint64_t checksum;   /* written by gpuos_ring_publish */
  double scalars[GPUOS_MAX_SCALARS];
  gpuos_view views[1 + GPUOS_MAX_INPUTS]; /* [0] = output */
  uint64_t reserved2[2];
} gpuos_task;

/* Completion cell (8 bytes in mapped pinned memory), written exactly once by
 * whoever finished the task.  On the worker path the completer issues a
 * gpu-scope release fence (fence.release.gpu, one per run of finished tasks)
 * and then a relaxed system-scope store of the word: outputs are in L2 -- the
 * point the host's copy engine and managed-memory migration read from --
 * before the word is posted.  A sys-scope fence is the formal PTX guarantee
 * for a host-CPU observer; it measured +3 us on the depth-1 p50 (8.3 -> 11.3
 * us) for no throughput change, so the gpu-scope fence is kept and this is
 * the documented assumption.  The per-op path uses
 * fence.acq_rel.sys.  Layout:
 *   bits 0..7 state (0 Pending, 1 Done, 2 Failed), bits 8..15 ErrorCode,
 *   bits 16..63 low 48 bits of the task seq.
 * Replaces HandleState (runtime.hpp:59-88). */
#define GPUOS_CELL_STATE(w) ((unsigned)((w)&0xffu))
#define GPUOS_CELL_CODE(w) ((int)(((w) >> 8) & 0xffu))

typedef struct gpuos_cfg {
  uint64_t capacity;          /* ring slots; rounded up to a power of two, min 2 (queue.hpp:162-172) */
  uint32_t table_slots;       /* operator table size (runtime.hpp:179); min 33 */
  uint32_t num_workers;       /* worker CTAs; 0 = one per SM */
  uint32_t threads_per_worker;/* CTA size (PAPER.md:303 threads_per_block); 0 = 256 */
  uint32_t spin_iterations;   /* polls before backoff (executor.hpp:29) */
  uint32_t backoff_max_exp;   /* nanosleep ladder 2^k * 64 ns (executor.hpp:30) */
  uint32_t telemetry;         /* device trace ring on/off (runtime.hpp:181) */
  uint64_t yield_every;       /* executor.hpp:28 */
  uint64_t trace_capacity;    /* device trace ring slots (runtime.hpp:180) */
  uint64_t flags;             /* GPUOS_CFG_* */
  uint64_t reserved[3];
} gpuos_cfg;

/* gpuos_cfg.flags: buffers in plain device memory (cudaMalloc) instead of
 * managed memory.  Faster host<->device copies (measured 1.34M vs 1.04M
 * config-1 e2e tasks/s); BufferPool::data<T>() pointers are then device
 * pointers, so host access goes through upload/download. */
#define GPUOS_CFG_DEVICE_BUFFERS 0x1ull
/* gpuos_cfg.flags: open without a resident generation (as env
 * GPUOS_DEFER_START=1): work published before gpuos_dev_run_finite is drained
 * by one finite generation, which profilers that serialise kernel launches
 * (ncu) can capture; gpuos_dev_start makes it persistent. */
#define GPUOS_CFG_DEFER_START 0x2ull

typedef struct gpuos_dev gpuos_dev; /* opaque per-GPU runtime */

typedef struct gpuos_snapshot { /* TaskQueue::Snapshot (queue.hpp:156-160) */
  uint64_t head;      /* tasks claimed by workers */
  uint64_t tail;      /* tasks published */
  uint64_t processed; /* tasks completed */
} gpuos_snapshot;

typedef struct gpuos_dev_stats {
  uint64_t processed;
  uint64_t failed;
  uint64_t canary_hits;
  uint64_t stalls;
  uint64_t torn_reads;
  uint64_t per_op[256];
} gpuos_dev_stats;

typedef struct gpuos_tracepoint { /* telemetry.hpp:22-32 */
  uint64_t seq;
  uint64_t op_id;
  uint32_t worker;
  uint32_t reserved;
  uint64_t enqueue_ns;
  uint64_t dequeue_ns;
  uint64_t exec_ns;
  uint64_t version;
} gpuos_tracepoint;

/* One stack-machine instruction of an injected elementwise operator
 * (reference bytecode.hpp:18-34 opcodes, same numbering). */
typedef struct gpuos_instr {
  uint8_t op;
  uint8_t pad[3];
  int32_t k;    /* LoadIn index; Narrow dtype */
  double value; /* PushConst payload */
} gpuos_instr;

enum gpuos_opcode {
  GPUOS_BC_PUSH_CONST = 0, GPUOS_BC_LOAD_IN, GPUOS_BC_ADD, GPUOS_BC_SUB, GPUOS_BC_MUL,
  GPUOS_BC_DIV, GPUOS_BC_NEG, GPUOS_BC_EXP, GPUOS_BC_TANH, GPUOS_BC_MAX, GPUOS_BC_MIN,
  GPUOS_BC_ABS, GPUOS_BC_SQRT, GPUOS_BC_NARROW, GPUOS_BC_STORE_OUT
};

#define GPUOS_MAX_PROGRAM 256 /* instructions per injected program */
#define GPUOS_MAX_STACK 32    /* device evaluation stack (verified bound) */

typedef struct gpuos_inject_stats {
  uint64_t upload_ns;   /* program upload to HBM */
  uint64_t epoch_wait_ns;
  uint64_t bank_write_ns;
  uint64_t flip_ns;
  uint64_t version;     /* table version published by the install */
} gpuos_inject_stats;

/* ---------------- lifecycle (Runtime ctor/dtor, Executor start/stop:
 *                   runtime.hpp:207-223, executor.hpp:72-128) ---------------- */
int gpuos_abi_version(void);
int gpuos_default_cfg(gpuos_cfg* cfg);
/* Allocate ring/table/device state on `device` and launch the persistent worker kernel. */
int gpuos_dev_open(int device, const gpuos_cfg* cfg, gpuos_dev** out);
/* Sentinel behind all published work, drain, join (executor.hpp:87-94), free everything. */
int gpuos_dev_close(gpuos_dev* dev);
/* 1 while the persistent kernel is resident (executor.hpp:101-102), else 0. */
int gpuos_dev_alive(gpuos_dev* dev);
/* Drain-then-stop the workers without freeing state; gpuos_dev_start relaunches them. */
int gpuos_dev_stop(gpuos_dev* dev);
int gpuos_dev_start(gpuos_dev* dev);
int gpuos_dev_num_workers(gpuos_dev* dev, uint32_t* n);
int gpuos_dev_sm_count(gpuos_dev* dev, uint32_t* n);
/* Hold (1) / release (0) ticket claims: idle workers stop claiming while held,
 * so published work stays queued (lets tests fill the ring; stop releases). */
int gpuos_dev_hold(gpuos_dev* dev, int hold);
/* With the workers stopped: publish the shutdown sentinel behind all queued
 * work, run one worker generation until it drains the ring and exits, and
 * report its duration (CUDA events on the worker stream).  A finite kernel
 * for ncu and for device-capacity measurements. */
int gpuos_dev_run_finite(gpuos_dev* dev, float* kernel_ms);
/* Live yield cadence (executor.hpp:107). */
int gpuos_set_yield_every(gpuos_dev* dev, uint64_t n);
/* Convert a device %globaltimer stamp to host steady_clock ns. */
int gpuos_dev_clock_offset(gpuos_dev* dev, int64_t* offset_ns);

/* ---------------- device memory (BufferPool, tensor.hpp:259-327) ---------------- */
/* Zero-filled, never-reused ids (tensor.hpp:267-278).  Storage is CUDA managed
 * memory so host pointers from BufferPool::data<T>() stay valid. */
int gpuos_buf_alloc(gpuos_dev* dev, int dtype, uint64_t n, uint64_t* id, void** ptr);
int gpuos_buf_free(gpuos_dev* dev, uint64_t id);
int gpuos_buf_lookup(gpuos_dev* dev, uint64_t id, int* dtype, uint64_t* n, void** ptr);
/* dir: 0 = host->device, 1 = device->host, 2 = device->device; synchronous on a side stream. */
int gpuos_buf_copy(gpuos_dev* dev, void* dst, const void* src, uint64_t bytes, int dir);
/* Fill `bytes` bytes at `dst` (buffer memory) with `byte` on the side stream,
 * synchronously.  Benchmarks poison outputs (0xff: NaN) before a verified
 * step so stale results cannot pass the check (BufferPool::fill). */
int gpuos_buf_fill(gpuos_dev* dev, void* dst, int byte, uint64_t bytes);
/* Migrate a buffer's pages to HBM ahead of a timed run. */
int gpuos_buf_prefetch(gpuos_dev* dev, uint64_t id);
/* Fill a view descriptor for buffer `id` (resolves addr, status, bounds). */
int gpuos_view_bind(gpuos_dev* dev, uint64_t id, int dtype, int64_t offset, int rank,
                    const int64_t* extents, const int64_t* strides, gpuos_view* out);

/* ---------------- completion cells (HandleState, runtime.hpp:59-88) ---------------- */
/* `count` cells of mapped pinned memory, zeroed (Pending).  *host is the host
 * view, *device_addr the address to place in gpuos_task.done_cell. */
int gpuos_cells_alloc(gpuos_dev* dev, uint64_t count, uint64_t** host, uint64_t* device_addr);

/* ---------------- task ring (TaskQueue, queue.hpp:154-301) ---------------- */
int gpuos_ring_capacity(gpuos_dev* dev, uint64_t* capacity);
/* Reserve the next position; QueueFull when the slot one lap down is unclaimed (queue.hpp:179-187). */
int gpuos_ring_reserve(gpuos_dev* dev, uint64_t* pos);
/* Publish into a reserved position: copy, checksum, release (queue.hpp:192-231). */
int gpuos_ring_publish(gpuos_dev* dev, uint64_t pos, const gpuos_task* task);
/* Dense submit fast path: every operand (output + n_inputs inputs) is a
 * row-major contiguous view of the same dtype and extents, bound in range,
 * with at most one scalar.  Reserve + publish in one call, straight into the
 * ring's compact encoding; QueueFull when the next slot is still in use.
 * Equivalent to gpuos_ring_reserve + gpuos_ring_publish of the gpuos_task
 * build_task would produce (queue.hpp:179-231). */
typedef struct gpuos_dense_task {
  uint64_t seq;
  uint64_t done_cell;
  uint64_t size;        /* output element count */
  uint32_t op_id;
  uint16_t flags;
  uint8_t n_inputs;
  uint8_t n_scalars;    /* 0 or 1 */
  uint8_t dtype;
  uint8_t rank;
  uint8_t reserved[6];
  int32_t extents[GPUOS_MAX_RANK];
  uint64_t addr[1 + GPUOS_MAX_INPUTS]; /* [0] = output */
  double scalar0;
  uint64_t wait_target; /* GPUOS_FLAG_AFTER: processed count to wait for */
} gpuos_dense_task;
int gpuos_ring_submit_dense(gpuos_dev* dev, const gpuos_dense_task* task);
/* Producer view of the ring for a header-side dense publisher: the caller's
 * thread writes compact slots itself (gdev::ring_write_dense in
 * include/gpuos_ring_format.h, the same code gpuos_ring_submit_dense runs),
 * saving the library call and the descriptor hand-off per task.  Single
 * producer: `reserve` is the cursor gpuos_ring_reserve/_submit_dense share. */
typedef struct gpuos_ring_view {
  char* ring;               /* cap x 128-byte slots (mapped pinned) */
  uint64_t mask;            /* cap - 1 */
  uint64_t cap;
  uint64_t* reserve;        /* producer cursor */
  uint64_t* tail;           /* published count, read by the device */
  const uint32_t* trace_on; /* enqueue stamps wanted */
} gpuos_ring_view;
int gpuos_ring_view_get(gpuos_dev* dev, gpuos_ring_view* out);

/* Monitoring snapshot; head <= tail always holds. */
int gpuos_ring_peek(gpuos_dev* dev, gpuos_snapshot* out);
/* Block until processed >= `count` (wait_all, runtime.hpp:399-406). */
int gpuos_ring_wait_processed(gpuos_dev* dev, uint64_t count);
/* One-line JSON of the ring cursors and device control words (diagnostics). */
int gpuos_dev_debug(gpuos_dev* dev, char* buf, size_t cap);

/* ---------------- operator table (OperatorTable, optable.hpp:98-251) ---------------- */
int gpuos_table_slots(gpuos_dev* dev, uint32_t* slots);
int gpuos_table_version(gpuos_dev* dev, uint64_t* version);
/* Entry status in the active bank: 0 Empty, 1 Active, 2 Killed (optable.hpp:40). */
int gpuos_table_status(gpuos_dev* dev, uint32_t op_id, int* status, int* kind);
/* Install a device task body: one version bump each (optable.hpp:126-131, 197-234). */
int gpuos_table_install_builtin(gpuos_dev* dev, uint32_t op_id, uint32_t kind);
/* Install an injected elementwise program (upload + dual-bank flip, no kernel restart). */
int gpuos_table_install_program(gpuos_dev* dev, uint32_t op_id, const gpuos_instr* code,
                                uint32_t n_instr, int arity, int dtype, gpuos_inject_stats* stats);
/* Upload a verified elementwise program for per-task use (fused composites):
 * returns its device address; programs live for the runtime's lifetime. */
int gpuos_program_upload(gpuos_dev* dev, const gpuos_instr* code, uint32_t n_instr, int arity, int dtype,
                         uint64_t* device_addr);
/* Fail-fast stub under a new version (optable.hpp:135-142). */
int gpuos_table_kill(gpuos_dev* dev, uint32_t op_id);

/* ---------------- telemetry (Counters/TraceRing, telemetry.hpp:22-196) ---------------- */
int gpuos_dev_get_stats(gpuos_dev* dev, gpuos_dev_stats* out);
int gpuos_trace_enable(gpuos_dev* dev, int on);
/* Copy up to `cap` most recent device tracepoints (oldest first), host clock. */
int gpuos_trace_snapshot(gpuos_dev* dev, gpuos_tracepoint* out, uint64_t cap, uint64_t* n);

/* Per-task phase stamps of the same records, all on the host steady clock:
 * commit, fetcher starts polling the ticket, publication observed, task
 * staged and resolved (dequeue), body finished, completion posted;
 * `reserved` = ns from dequeue until the executor group picked it up. */
typedef struct gpuos_trace_phase {
  uint64_t seq;
  uint64_t enqueue_ns;
  uint64_t ticket_ns;
  uint64_t seen_ns;
  uint64_t dequeue_ns;
  uint64_t end_ns;
  uint64_t done_ns;
  uint32_t worker;
  uint32_t reserved;
} gpuos_trace_phase;
int gpuos_trace_phases(gpuos_dev* dev, gpuos_trace_phase* out, uint64_t cap, uint64_t* n);

/* ---------------- conventional path / baseline (a) ---------------- */
/* One cudaLaunchKernel of the same task body as a standalone kernel
 * (execute_inline, runtime.hpp:567-619).  `stream` is a cudaStream_t or NULL
 * for the runtime's side stream.  The body writes task->done_cell. */
int gpuos_launch_task(gpuos_dev* dev, const gpuos_task* task, void* stream);
/* Lean per-op baseline (measurement only, not a task path): one launch of a
 * minimal dense f32 add kernel -- 4 small parameters, no descriptor, no dynamic
 * shared memory, no table lookup, no lock.  The caller owns the device's
 * current context; pointers must be 16-byte aligned. */
int gpuos_launch_lean_add(gpuos_dev* dev, void* out, const void* a, const void* b, int64_t n, void* stream);
int gpuos_stream_create(gpuos_dev* dev, void** stream);
int gpuos_stream_sync(gpuos_dev* dev, void* stream);
int gpuos_stream_destroy(gpuos_dev* dev, void* stream);

/* ---------------- timing and host staging (bench / e2e) ---------------- */
/* The stream the persistent worker kernel is launched on.  An event recorded
 * there before gpuos_dev_start and another after it completes when the
 * worker kernel exits, so a pair brackets one kernel lifetime. */
int gpuos_dev_kernel_stream(gpuos_dev* dev, void** stream);
int gpuos_event_create(gpuos_dev* dev, void** event);
int gpuos_event_record(gpuos_dev* dev, void* event, void* stream);
int gpuos_event_sync(gpuos_dev* dev, void* event);
/* 1 when all work before the event has completed, 0 while pending (non-blocking). */
int gpuos_event_done(gpuos_dev* dev, void* event);
int gpuos_event_elapsed_ms(gpuos_dev* dev, void* start, void* stop, float* ms);
int gpuos_event_destroy(gpuos_dev* dev, void* event);
/* Pinned host staging memory (freed at gpuos_dev_close). */
int gpuos_host_alloc(gpuos_dev* dev, uint64_t bytes, void** ptr);
/* dir as gpuos_buf_copy; enqueued on `stream` (NULL = side stream), not synchronised. */
int gpuos_copy_async(gpuos_dev* dev, void* dst, const void* src, uint64_t bytes, int dir, void* stream);

/* ---------------- NVRTC / nvJitLink (ModuleCache compile step, opcompiler.hpp:180-189) ---------------- */
/* Compile CUDA source to a relocatable sm_100a cubin and link it with nvJitLink.
 * Buffers are malloc'd; free with gpuos_free.  Timings in ns. */
int gpuos_jit_compile(const char* src, const char* const* opts, int nopts, void** cubin,
                      size_t* size, uint64_t* compile_ns, uint64_t* link_ns, char* log, size_t logcap);
void gpuos_free(void* p);

/* ---------------- natively compiled injected operators ----------------
 * The live injection path installs a verified device program (no module load,
 * no kernel restart).  Promotion to native code: the op's program is turned
 * into CUDA C++ by the host runtime, compiled by NVRTC to a relocatable
 * sm_100a object, linked by nvJitLink with the relocatable worker image into
 * a new worker module, and loaded at a generation handover (drain at a ticket
 * boundary, load, relaunch; cuModuleLoadData blocks while a kernel is
 * resident).  The table entry then names a native kind with the program kept
 * as fallback (ModuleCache compile step, opcompiler.hpp:180-189). */
#define GPUOS_NATIVE_SLOTS 32 /* natively compiled injected ops per device */
typedef struct gpuos_native_stats {
  uint64_t drain_ns;    /* sentinel published -> resident generation exited */
  uint64_t load_ns;     /* cuModuleLoadData + symbol lookup + jit table write */
  uint64_t relaunch_ns; /* new generation launched */
} gpuos_native_stats;
int gpuos_jit_compile_object(const char* src, void** obj, size_t* size, uint64_t* compile_ns, char* log,
                             size_t logcap);
int gpuos_jit_link_worker(const void* const* objs, const size_t* sizes, int n, void** cubin, size_t* size,
                          uint64_t* link_ns, char* log, size_t logcap);
/* `ptr_syms[i]` names a __device__ function-pointer variable of the module
 * holding the native op for jit slot `slots[i]`. */
int gpuos_dev_load_native(gpuos_dev* dev, const void* cubin, size_t size, const uint32_t* slots,
                          const char* const* ptr_syms, int n, gpuos_native_stats* stats);
/* Like gpuos_table_install_program, but the entry dispatches native jit slot
 * `slot` (the program stays attached as the fallback body). */
int gpuos_table_install_native(gpuos_dev* dev, uint32_t op_id, uint32_t slot, const gpuos_instr* code,
                               uint32_t n_instr, int arity, int dtype, gpuos_inject_stats* stats);

/* Human-readable name of an error code (errors.hpp:43-72). */
const char* gpuos_error_name(int code);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* GPUOS_CUDA_H_ */
