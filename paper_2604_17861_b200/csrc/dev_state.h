// Layout shared by the host runtime (capi.cu) and the device worker
// (worker.cu): device-resident control state, the dual-bank operator table
// entry, the device trace record, and the launch helpers worker.cu exports.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "gpuos_cuda.h"

namespace gdev {

constexpr uint32_t kMaxWorkers = 2048;
constexpr uint64_t kQuiescent = ~0ull;  // EpochRegistry::kQuiescent (optable.hpp:62)
constexpr uint64_t kRunning = ~0ull;    // stop_pos while running
constexpr uint32_t kNumKinds = 80;      // module jump-table slots
// Natively compiled injected operators (NVRTC + nvJitLink, linked into a
// worker module at a generation handover): kinds [kJitKindBase, +kJitSlots)
// dispatch through DevState::jit_fns; a generation without that code falls
// back to the entry's device program (TableEntry::aux).
constexpr uint32_t kJitKindBase = 96;
constexpr uint32_t kJitSlots = 32;
constexpr uint32_t kTaskBytes = 384;
constexpr uint32_t kCtlBytes = 128;     // per-task control block (standalone kernels)
constexpr uint32_t kHeaderBytes = 8192;  // worker: task buffers, control blocks, counters, entry cache
constexpr uint32_t kScratchBytes = 91 * 1024;
constexpr uint32_t kLaunchCounters = 1u << 16;

// One operator-table entry (optable.hpp:40-48): the device function is named
// by `kind`, an index into the loaded module's jump table, so a bank image
// stays valid across worker-kernel generations.
struct TableEntry {
  uint16_t kind;
  uint8_t status;  // 0 Empty, 1 Active, 2 Killed
  uint8_t pad[5];
  uint64_t aux;    // program pointer for GPUOS_KIND_PROGRAM
};
static_assert(sizeof(TableEntry) == 16, "table entry is 16 bytes");

// Injected-program image in HBM: header then n_instr gpuos_instr.
struct ProgramHeader {
  uint32_t n_instr;
  int32_t arity;
  int32_t dtype;
  int32_t max_stack;
};

typedef void* OpFn_;  // device function pointer (OpFn) as stored in HBM

struct TraceRec {  // Tracepoint (telemetry.hpp:22-32) plus a publication stamp
  uint64_t stamp;  // ticket*2+2 once complete
  uint64_t seq;
  uint64_t op_id;
  uint64_t worker;
  uint64_t enqueue_ns;  // host clock (copied from the descriptor)
  uint64_t dequeue_gt;  // device %globaltimer at claim
  uint64_t exec_ns;
  uint64_t version;
  uint64_t t_ticket;  // phase stamps (%globaltimer): ticket taken,
  uint64_t t_seen;    //   publication observed,
  uint64_t t_done;    //   completion posted
  uint64_t pad;
};

struct alignas(128) DevState {
  // hot words on private 128-byte lines
  uint64_t claim;      // ticket cursor (atomicAdd by claiming warps)
  uint64_t pad0[15];
  uint64_t hint;       // highest producer tail observed on the device
  uint64_t pad1[15];
  uint64_t version;    // operator-table version (optable.hpp:476)
  uint64_t pad2[15];
  uint64_t stop_pos;   // position of the consumed shutdown sentinel, kRunning otherwise
  uint64_t yield_every;
  uint32_t trace_on;
  uint32_t spin_iterations;
  uint32_t backoff_max_exp;
  uint32_t hold;       // nonzero: idle workers take no new ticket (test/handover hook)
  uint64_t pad3[12];
  // device counters (Counters, telemetry.hpp:142-196)
  uint64_t processed;
  uint64_t failed;
  uint64_t canary_hits;
  uint64_t stalls;
  uint64_t torn_reads;
  uint64_t trace_head;
  uint64_t pad4[10];
  uint64_t per_op[256];
  // operator table: two banks selected by version parity (optable.hpp:98-104)
  TableEntry* bank[2];
  uint64_t bank_gen[2];  // generation stamped on every entry of a bank image
  uint32_t table_slots;
  uint32_t num_workers;
  // task ring in mapped pinned host memory
  const char* ring;  // cap x kRingSlot (ring_format.h)
  const char* ext;   // cap x kExtBytes
  uint64_t cap;
  uint64_t mask;
  const uint64_t* host_tail;  // producer's published count
  uint64_t* host_done;        // per-worker processed counts (device-written)
  uint64_t* host_claimed;     // per-worker claimed counts
  uint64_t* host_epoch;       // per-worker published table epoch
  uint64_t* dev_epoch;        // same, in HBM
  TraceRec* trace;
  uint64_t trace_cap;
  OpFn_* jit_fns;  // kJitSlots entries, filled by the host after loading a native module (null = none)
};

#ifndef __CUDACC_RTC__
// ---- host-callable helpers implemented in worker.cu ----
void load_all_kernels(int* worker_regs, size_t* worker_local);
cudaError_t launch_worker(DevState* s, uint32_t workers, uint32_t threads, uint32_t smem, cudaStream_t st);
cudaError_t launch_task(const gpuos_task* t, uint32_t kind, uint64_t aux, uint32_t nparts,
                        uint32_t* counter, cudaStream_t st);
cudaError_t launch_clock_probe(const uint32_t* flag, uint64_t* out, int rounds, cudaStream_t st);
// Stream-ordered generation start: claim/hint/stop_pos in one tiny launch
// (three pageable 8-byte copies cost more stream time than the launch).
cudaError_t launch_lean_add(float* out, const float* a, const float* b, int n, cudaStream_t st);
cudaError_t launch_gen_init(DevState* s, uint64_t claim, uint64_t hint, uint64_t stop_pos, cudaStream_t st);
uint32_t worker_smem_bytes();
uint32_t worker_threads();
int smem_carveout();  // preferred shared carveout (percent) for every kernel, GPUOS_CARVEOUT overrides
cudaError_t worker_occupancy(int* per_sm);

#endif  // __CUDACC_RTC__

}  // namespace gdev
