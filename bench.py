#!/usr/bin/env python3
"""Benchmark: small-op tasks/s through the persistent B200 GPUOS runtime.

Workload (BASELINE.json metric, configs[0]/[1] headline): one step = 10,000
fp32 Add tasks of 4,096 contiguous elements on one task ring with the builtin
table, distinct a_i/b_i/c_i per task (491.5 MB working set, > 126 MB L2),
submitted through gpuos::Runtime::submit.  A step launches the persistent
worker kernel, submits every task, waits, and retires the kernel with the
shutdown sentinel; its duration is measured with CUDA events bracketing the
worker kernel on its own stream.  ``value`` = tasks of all ranks / max-over-
ranks time.  Also reported: baseline (a) one cudaLaunchKernel per task, queue-
depth-1 submit->complete latency, the e2e arm (inputs and outputs in pinned
host memory, copies in the timed region), the roofline of the worker kernel,
the reference CPU implementation (oracle/_ref) timed on the host cores, and
SM clocks sampled during the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
LIBDIR = os.path.join(ROOT, "paper_2604_17861_b200", "lib")
METRIC = "small-op tasks/sec and p50 submit-to-complete µs (4K-elem fp32 ops), 1-8 B200"
N_TASKS, N_ELEMS = 10_000, 4096
BYTES_PER_TASK = N_ELEMS * 12  # 2 x 16 KiB read + 16 KiB write
WORKLOAD = ("config1: 10,000 fp32 Add tasks x 4096 contiguous elements per step, one task ring, "
            "builtin op table, distinct buffers per task")


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every 2 ms while
    the timed region runs (the recipe's nvidia-smi clocks line, in-process so
    that millisecond-scale regions still get samples)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm: list[float] = []
        self.max_sm = None
        self.reasons: set[str] = set()
        self.stop_flag = threading.Event()
        self.thread = None
        self.err = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_flag.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception as e:  # noqa: BLE001
                self.err = str(e)
                return
            time.sleep(0.002)

    def stop(self) -> dict:
        self.stop_flag.set()
        if self.thread:
            self.thread.join(timeout=2)
        if self.err and not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err]}
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_sm,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


def launch_replicas(n_gpus: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks of this script
    (one process per GPU, torchrun's env contract, rendezvous on 127.0.0.1)
    and relay rank 0's line.  Under torchrun RANK is already set."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n_gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n_gpus), LOCAL_WORLD_SIZE=str(n_gpus),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=subprocess.PIPE if r == 0 else subprocess.DEVNULL))
    out = procs[0].communicate()[0].decode()
    rc = max(p.wait() for p in procs)
    sys.stdout.write(out)
    return rc


def dist_setup(n_gpus: int):
    if n_gpus <= 1 or "RANK" not in os.environ:
        return None, 0, 1, 0
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group(backend="gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    return dist, rank, world, local


def dist_max(dist, x: float) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier(dist):
    if dist is not None:
        dist.barrier()


def dist_gather(dist, x: float) -> list:
    """Every rank's value of x (rank order)."""
    if dist is None:
        return [x]
    import torch
    out = [torch.zeros(1, dtype=torch.float64) for _ in range(dist.get_world_size())]
    dist.all_gather(out, torch.tensor([x], dtype=torch.float64))
    return [float(t.item()) for t in out]


def dist_sum(dist, x: float) -> float:
    return sum(dist_gather(dist, x))


ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")


def load_checker(lib) -> bool:
    """Parity leg: hand the oracle (test-only CPU restatement, pinned to the
    reference by tests/) to the bench library as the checker.  It runs only
    after timed regions, on outputs poisoned before the verified step."""
    lib.gb_set_oracle.argtypes = [C.c_char_p]
    return os.path.exists(ORACLE_SO) and lib.gb_set_oracle(ORACLE_SO.encode()) == 0


def ref_cpu_baseline(seconds: float, steps: int = 0) -> dict | None:
    """The reference gpuos::Runtime (built from /root/reference into oracle/_ref)
    on the host cores: config-1 steps of 10,000 add tasks, all host threads."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    cmd = [exe, "--tasks", str(N_TASKS), "--elems", str(N_ELEMS), "--seconds", str(seconds)]
    if steps:
        cmd += ["--steps", str(steps)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    for line in out.stdout.splitlines():
        if line.startswith("{"):
            return json.loads(line)
    return None


def run_reference(args) -> None:
    dist, rank, world, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    res = ref_cpu_baseline(seconds=0, steps=args.steps + args.warmup)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_bench not built"}))
        return
    timed = res["step_seconds"][args.warmup:]
    tot = sum(timed)
    value = N_TASKS * len(timed) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tasks/s", "n_gpus": args.gpus,
        "steps": len(timed), "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "tasks_per_step": N_TASKS, "elems": N_ELEMS,
                   "parallelism": "host threads (reference worker pool)"},
        "cpu_baseline": {"value": value, "unit": "tasks/s", "cores": res["workers"], "kind": "reference",
                         "sample": f"{len(timed)} steps x {N_TASKS} tasks x {N_ELEMS} fp32 adds"},
        "e2e": {"value": value, "unit": "tasks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "p50_submit_to_complete_us": res.get("p50_us"),
    }
    print(json.dumps(line))


def parity_dict(vals, checked_what: str) -> dict:
    """[mismatched tasks, checked tasks, checked elements, float-sum bit-exact
    share, mismatched elements] from the bench library (put_tally)."""
    if vals[0] < 0:
        return {"checked": 0, "note": "no checker (oracle/liboracle.so missing)"}
    return {"mismatches": int(vals[0]), "checked": int(vals[1]), "checked_elements": int(vals[2]),
            "float_sum_bitexact_frac": vals[3], "mismatched_elements": int(vals[4]), "what": checked_what}


def run_config5(lib, dist, rank: int, world: int, local: int, tasks_per_stream: int, streams: int = 8) -> dict:
    """Config 5: `streams` independent config-2 streams, stream s on GPU s mod G
    (G = world); every rank builds its streams, a barrier, then all ranks run
    their streams concurrently; device time = max over ranks of each rank's
    union of worker-kernel lifetimes.  At G > 1 the same streams also run at
    G = 1 (all on rank 0's GPU) for rate(G) / (G * rate(1))."""
    peaks = load_peaks()
    lib.gb_c5_open.restype = C.c_void_p
    lib.gb_c5_open.argtypes = [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_longlong]
    lib.gb_c5_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_c5_survivors.argtypes = [C.c_void_p]
    lib.gb_c5_survivors.restype = C.c_double
    lib.gb_c5_close.argtypes = [C.c_void_p]
    out_cap = 1 << 27  # output-ring elements per dtype per stream

    def run(g: int, active: bool, verify: int):
        mine = [s for s in range(streams) if s % g == rank] if active else []
        n = len(mine)
        res = (C.c_double * 16)()
        h = None
        if n:
            workers = max(1, 148 // n)
            ids = (C.c_int * n)(*mine)
            h = lib.gb_c5_open(local, ids, n, tasks_per_stream, workers, out_cap)
        dist_barrier(dist)
        if h:
            lib.gb_c5_run(h, 1, verify, res)
        ms = res[1] if n else 0.0
        surv = lib.gb_c5_survivors(h) if h else 0.0
        if h:
            lib.gb_c5_close(h)
        tot_ms = dist_max(dist, ms)
        tasks = dist_sum(dist, res[0] if n else 0.0)
        byts = dist_sum(dist, res[2] if n else 0.0)
        failed = dist_sum(dist, res[3] if n else 0.0)
        par = [dist_sum(dist, res[4 + i] if n else 0.0) for i in (0, 1, 2)] + [0.0]
        par.append(dist_sum(dist, res[8] if n else 0.0))
        se = dist_sum(dist, res[2 + 4] * res[3 + 4] if n else 0.0)  # bit-exact share, element-weighted
        par[3] = se / par[2] if par[2] else 1.0
        if not verify:
            par = [-1.0] * 5
        per_rank_ms = dist_gather(dist, ms)
        surv_all = dist_sum(dist, surv)
        return {"tasks": tasks, "ms": tot_ms, "bytes": byts, "failed": failed, "parity": par,
                "per_rank_ms": per_rank_ms, "survivors": surv_all, "submit_ns": res[9] if n else 0.0}

    r = run(world, True, 1)
    g = world
    rate = r["tasks"] / (r["ms"] / 1e3)
    gbps = r["bytes"] / (r["ms"] / 1e3) / 1e9
    res = {
        "workload": f"{streams} independent config-2 streams (seeds 42..{41 + streams}) x {tasks_per_stream:,} mixed "
                    f"micro-ops, stream s on GPU s mod G (G={g}), one host producer thread and one runtime (ring + "
                    f"persistent generation of {148 // max(1, -(-streams // g))} CTAs) per stream; device time = union "
                    "of the streams' worker-kernel lifetimes, max over GPUs",
        "G": g, "tasks_per_s": rate, "alg_GBps": gbps,
        "roofline_frac_per_gpu": gbps / (g * peaks["hbm_gbs"]), "failed_tasks": int(r["failed"]),
        "union_ms": r["ms"], "per_gpu_ms": r["per_rank_ms"], "host_submit_ns_per_task": r["submit_ns"],
        "parity": parity_dict(r["parity"], f"surviving outputs of the output rings ({int(r['survivors']):,} of "
                                           f"{int(r['tasks']):,} tasks; each output region is reused every "
                                           f"{out_cap:,} elements of its dtype)"),
    }
    if g > 1:
        r1 = run(1, rank == 0, 0)
        rate1 = r1["tasks"] / (r1["ms"] / 1e3)
        res["rate_G1_tasks_per_s"] = rate1
        res["scaling_efficiency"] = rate / (g * rate1)
    return res


def run_configs(lib, local: int, tasks2: int, tasks5: int) -> dict:
    """BASELINE.json configs 2-4 on this GPU (tools/bench/gpuos_bench_configs.cpp),
    each verified against the oracle after its timed steps."""
    peaks = load_peaks()
    lib.gb_config2.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_config3.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_config4.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    out = (C.c_double * 32)()
    res = {}
    lib.gb_config2(local, tasks2, 3, out)
    res["config2_mixed"] = {
        "workload": "mixed {add,mul,relu,reduce_sum} x {f32,f16,bf16,i32}, numel log-uniform 64..65536, "
                    f"contiguous/strided/broadcast layouts, seed 42; {tasks2:,} tasks per step, distinct outputs",
        "tasks_per_s": out[0], "alg_GBps": out[1], "roofline_frac": out[1] / peaks["hbm_gbs"],
        "mean_bytes_per_task": out[3], "failed_tasks": int(out[4]), "host_submit_ns_per_task": out[5],
        "parity": parity_dict(list(out[6:11]), "every task of the last timed step (outputs poisoned before it)")}
    for name, dt in (("config3_attention_f32", 0), ("config3_attention_bf16", 4)):
        lib.gb_config3(local, dt, 20, out)
        res[name] = {
            "workload": "32 heads x seq 128 x head_dim 64: Q*scale, Q.K^T (transposed view), softmax, P.V as "
                        "128 individual tasks per step, host waits between the 4 phases",
            "step_us": out[0], "tasks_per_s": out[1], "gflops": out[2], "failed_tasks": int(out[3]),
            "max_rel_err": out[4],
            "phase_us": {"scale": out[5], "qk_t": out[6], "softmax": out[7], "pv": out[8]},
            "parity": parity_dict(list(out[9:14]), "all 32 heads x 4 phases of the last step vs the oracle on "
                                                   "that phase's GPU inputs")}
    # device-dependency variant: phases ordered on the device (Runtime::fence), one host wait per step
    lib.gb_config3_fenced.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for name, dt in (("config3_attention_f32_fenced", 0), ("config3_attention_bf16_fenced", 4)):
        lib.gb_config3_fenced(local, dt, 20, out)
        res[name] = {
            "workload": "config 3 with the 4 phases ordered on the device by Runtime::fence() (tasks of a phase "
                        "wait on the device's processed count for the previous phase) and one host wait per step",
            "step_us": out[0], "tasks_per_s": out[1], "gflops": out[2], "failed_tasks": int(out[3]),
            "max_rel_err": out[4],
            "parity": parity_dict(list(out[9:14]), "all 32 heads x 4 phases of the last step vs the oracle on "
                                                   "that phase's GPU inputs")}
    lib.gb_config4(local, 1_000_000, out)
    res["config4_hot_swap"] = {
        "workload": "1,000,000 fp32 4096-element tasks alternating builtin add and injected scale_add(1.5,-0.25); "
                    "scale_add re-injected as (-2,3) at task 500,000 with the 4096-slot ring full (streaming "
                    "reading of '1M in flight')",
        "tasks_per_s": out[0], "inject_call_ms": out[1],
        "swap_phases_us": {"upload": out[2], "epoch_wait": out[3], "bank_write": out[4], "flip": out[5]},
        "window_rows_checked": int(out[6]), "rows_not_one_variant": int(out[7]),
        "old_rows_past_window": int(out[8]), "failed_tasks": int(out[9]), "canary_hits": int(out[10]),
        "old_rows": int(out[11]), "new_rows": int(out[12])}
    lib.gb_swap_latency.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_swap_latency(local, 200_000, 16, out)
    res["config4_swap_latency"] = {
        "workload": "200,000 fp32 4096-element tasks alternating add and injected scale_add, re-injected 16 times "
                    "with the ring busy; device trace on",
        "entry_to_first_new_dispatch_us_p50": out[0], "entry_to_first_new_dispatch_us_max": out[1],
        "call_return_to_first_new_dispatch_us_p50": out[2], "inject_call_us_p50": out[3],
        "swaps_measured": int(out[4]), "old_version_dispatches_after_return_max": int(out[5]),
        "stream_tasks_per_s": out[6],
        "clock": "device dequeue stamps converted to the host steady clock (ping-pong calibration, +-1 us)"}
    lib.gb_native.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_native(local, 200_000, out)
    res["config4_native_promotion"] = {
        "workload": "200,000 fp32 4096-element scale_add(1.5,-0.25) tasks as a device program, then promoted to "
                    "native code (NVRTC -> relocatable sm_100a -> nvJitLink with the worker image -> module load at a "
                    "generation handover) and run again",
        "program_tasks_per_s": out[0], "native_tasks_per_s": out[1],
        "promotion_ms": {"codegen": out[2], "nvrtc": out[3], "nvjitlink": out[4]},
        "handover_us": {"drain": out[5], "module_load": out[6], "relaunch": out[7], "table_flip": out[8]},
        "output_mismatches_native_vs_program": int(out[9])}
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--capacity", type=int, default=4096)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the BASELINE configs 2-5 lines")
    ap.add_argument("--config2-tasks", type=int, default=1_000_000)
    ap.add_argument("--config5-tasks", type=int, default=1_000_000, help="tasks per stream")
    args = ap.parse_args()
    if args.gpus > 1 and "RANK" not in os.environ:
        sys.exit(launch_replicas(args.gpus))
    if args.impl == "reference":
        run_reference(args)
        return
    args.warmup = max(args.warmup, 3)

    dist, rank, world, local = dist_setup(args.gpus)
    lib_path = os.path.join(LIBDIR, "libgpuos_bench.so")
    if not os.path.exists(lib_path):
        raise SystemExit("libgpuos_bench.so not built: run __graft_entry__.build()")
    lib = C.CDLL(lib_path)
    checker = load_checker(lib)
    lib.gb_open.restype = C.c_void_p
    lib.gb_open.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
    lib.gb_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
    lib.gb_latency.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.gb_verify.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int]
    lib.gb_poison.argtypes = [C.c_void_p]
    lib.gb_checker.argtypes = [C.c_void_p]
    lib.gb_info.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
    lib.gb_close.argtypes = [C.c_void_p]

    h = lib.gb_open(local, N_TASKS, N_ELEMS, args.workers, args.capacity)
    out = (C.c_double * 8)()

    def step(mode):
        rc = lib.gb_step(h, mode, out)
        assert rc == 0
        return out[0], out[1], out[4], out[5]

    for _ in range(args.warmup):
        step(0)
    dev_ms, host_ms, sub_ms, fallbacks = [], [], [], 0
    bad_total, checked_total = 0, 0
    bad, checked = C.c_uint64(), C.c_uint64()
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.steps):
        # outputs poisoned (NaN) before every timed step and checked after it,
        # both outside the CUDA-event-timed worker-kernel lifetime
        lib.gb_poison(h)
        dist_barrier(dist)
        d, hm, fb, sm = step(0)
        dev_ms.append(d)
        host_ms.append(hm)
        sub_ms.append(sm)
        fallbacks += int(fb)
        lib.gb_verify(h, C.byref(bad), C.byref(checked), 0)
        bad_total += bad.value
        checked_total += checked.value
    clk = clocks.stop()
    dist_barrier(dist)
    total_dev_s = dist_max(dist, sum(dev_ms) / 1e3)
    total_host_s = dist_max(dist, sum(host_ms) / 1e3)
    per_rank_ms = dist_gather(dist, 1e3 * sum(dev_ms) / 1e3 / args.steps)
    bad_all = dist_sum(dist, float(bad_total))
    checked_all = dist_sum(dist, float(checked_total))

    # baseline (a): one cudaLaunchKernel per task, same bodies
    base_steps = max(1, min(args.steps, 3))
    step(1)  # warm
    b_dev = [step(1)[0] for _ in range(base_steps)]
    lean_dev = [step(3)[0] for _ in range(base_steps)]  # lean per-op launches (minimal add kernel)
    # queue-depth-1 latency, persistent vs per-op launch
    lat = (C.c_double * 3)()
    lib.gb_latency(h, 0, 10_000, 1_000, lat)
    p50, p99 = lat[0], lat[1]
    lib.gb_latency(h, 1, 2_000, 200, lat)
    lp50, lp99 = lat[0], lat[1]
    # e2e arm: host buffers, copies inside the timed region (host outputs
    # poisoned before every step, checked after the last)
    step(2)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        lib.gb_poison(h)
        e2e_ms.append(step(2)[1])
    e_bad, e_checked = C.c_uint64(), C.c_uint64()
    lib.gb_verify(h, C.byref(e_bad), C.byref(e_checked), 1)
    e2e_rate = N_TASKS / (statistics.median(e2e_ms) / 1e3)
    e2e_total = dist_sum(dist, e2e_rate)  # independent replicas: rates add
    info = C.create_string_buffer(512)
    lib.gb_info(h, info, 512)
    oracle_checked = bool(lib.gb_checker(h))
    lib.gb_close(h)
    configs = None
    if not args.no_configs:
        if world == 1:
            configs = run_configs(lib, local, args.config2_tasks, args.config5_tasks)
        else:
            configs = {"note": "configs 2-4 are single-GPU workloads, measured at --gpus 1"}
        c5 = run_config5(lib, dist, rank, world, local, args.config5_tasks)
        if rank == 0:
            configs["config5_streams"] = c5

    if rank != 0:
        dist_barrier(dist)
        return
    tasks_total = N_TASKS * args.steps * world
    value = tasks_total / total_dev_s
    per_step_dev_ms = 1e3 * total_dev_s / args.steps
    peaks = load_peaks()
    achieved_gbs = (N_TASKS * BYTES_PER_TASK) / (per_step_dev_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "worker_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get("bytes_per_step")
    base_value = N_TASKS / (statistics.median(b_dev) / 1e3)
    lean_value = N_TASKS / (statistics.median(lean_dev) / 1e3)
    cpu = None
    if not args.no_cpu_baseline:
        r = ref_cpu_baseline(seconds=args.cpu_seconds)
        if r is not None:
            cpu = {"value": r["tasks_per_s"], "unit": "tasks/s", "cores": r["workers"], "kind": "reference",
                   "sample": f"{r['tasks']} config-1 add tasks x {N_ELEMS} fp32 ({r['seconds']:.1f} s)"}
    line = {
        "metric": METRIC, "value": value, "unit": "tasks/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step_dev_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "tasks_per_step": N_TASKS, "elems": N_ELEMS, "global_batch": N_TASKS * world,
                   "l2": "inputs larger than L2 (491.5 MB distinct buffers per step; outputs poisoned between steps)",
                   "buffers": "device memory (RuntimeConfig::device_buffers); e2e copies pinned host <-> device",
                   "parallelism": f"independent ring + persistent kernel per GPU x{world}",
                   "runtime": json.loads(info.value.decode())},
        "per_gpu_ms_per_step": per_rank_ms,
        "p50_submit_to_complete_us": p50, "p99_submit_to_complete_us": p99,
        "host_clock_tasks_per_s": tasks_total / total_host_s,
        "host_submit_ns_per_task": 1e6 * statistics.median(sub_ms) / N_TASKS,
        "baseline_per_op_launch": {"value": base_value, "unit": "tasks/s", "p50_launch_sync_us": lp50,
                                   "p99_launch_sync_us": lp99, "speedup": value / (base_value * world)},
        "baseline_per_op_launch_lean": {
            "value": lean_value, "unit": "tasks/s", "speedup": value / (lean_value * world),
            "what": "one cudaLaunchKernel per task of a minimal dense f32 add kernel (4 parameters, no "
                    "descriptor, no dynamic shared memory, no lock, grid sized to the op), device-timed"},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved_gbs / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peaks["source"],
                     "kernel": "gpuos_worker_kernel (per step: 10,000 x 49,152 algorithmic bytes, slowest GPU)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_total, "unit": "tasks/s", "h2d_bytes_per_step": 2 * N_TASKS * N_ELEMS * 4 * world,
                "d2h_bytes_per_step": N_TASKS * N_ELEMS * 4 * world},
        "gpu_launches": args.steps * world,
        "parity": {"mismatches": int(bad_all), "checked": int(checked_all), "e2e_mismatches": e_bad.value,
                   "e2e_checked": e_checked.value,
                   "what": "every output element of every timed step (poisoned before the step) vs the "
                           + ("oracle's add" if oracle_checked else "host f32(a + b) (oracle not loaded: "
                                                                   "oracle/liboracle.so missing)")},
        "checker": "oracle/liboracle.so" if checker else None,
        "queue_full_fallbacks": fallbacks,
        "configs": configs,
        "clocks": clk,
    }
    print(json.dumps(line))
    dist_barrier(dist)


if __name__ == "__main__":
    main()
