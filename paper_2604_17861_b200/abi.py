"""ctypes binding of the C-ABI in include/gpuos_cuda.h.

This is the reference-side binding a Python maintainer would add (see
INTEGRATION.md); the parity tests and ``__graft_entry__.smoke()`` drive the
GPU path through it.  Loading fails loudly when ``libgpuos_cuda.so`` has not
been built: there is no CPU fallback behind this module.
"""
from __future__ import annotations

import ctypes as C
import os
import time
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libgpuos_cuda.so")

# ---- constants mirrored from gpuos_cuda.h ----
F32, F64, I32, F16, BF16 = 0, 1, 2, 3, 4
DTYPE_WIDTH = {F32: 4, F64: 8, I32: 4, F16: 2, BF16: 2}
DTYPE_NAMES = {F32: "f32", F64: "f64", I32: "i32", F16: "f16", BF16: "bf16"}
MAX_INPUTS, MAX_SCALARS, MAX_RANK = 4, 8, 4
SLOT_BYTES = 384
FLAG_FUSED, FLAG_SHUTDOWN, FLAG_UNCAPPED = 0x1, 0x2, 0x4
CFG_DEVICE_BUFFERS, CFG_DEFER_START = 0x1, 0x2
KIND_PROGRAM, KIND_KILLED = 64, 65
FIRST_INJECTED_ID = 32

OP = dict(add=0, mul=1, relu=2, gelu=3, softmax=4, layernorm=5, reduce_sum=6, reduce_max=7,
          reduce_min=8, matmul_small=9, vecmat=10, sdpa=11, rope=12, kv_append=13)

ERRORS = ["Ok", "IncompatibleShapes", "OutOfBounds", "InvalidBuffer", "ZeroCapacity", "QueueFull",
          "ZeroSlots", "OutOfRange", "NotInstalled", "OperatorKilled", "TableFull", "SyntaxError",
          "UnknownIdentifier", "ArityError", "VerifyError", "EmptyAxis", "DTypeMismatch",
          "ShapeMismatch", "TooLarge", "OddDim", "CacheFull", "AlreadyStarted", "RuntimeStopped",
          "IoError", "Internal"]
ERR = {name: i for i, name in enumerate(ERRORS)}

BC = dict(PUSH_CONST=0, LOAD_IN=1, ADD=2, SUB=3, MUL=4, DIV=5, NEG=6, EXP=7, TANH=8, MAX=9, MIN=10,
          ABS=11, SQRT=12, NARROW=13, STORE_OUT=14)


class View(C.Structure):
    _fields_ = [("addr", C.c_uint64), ("extents", C.c_int32 * 4), ("strides", C.c_int32 * 4),
                ("dtype", C.c_uint8), ("rank", C.c_uint8), ("status", C.c_uint8),
                ("reserved", C.c_uint8), ("buffer_lo", C.c_uint32)]


class Task(C.Structure):
    _fields_ = [("pub", C.c_uint64), ("seq", C.c_uint64), ("op_id", C.c_uint32), ("flags", C.c_uint16),
                ("n_inputs", C.c_uint8), ("n_scalars", C.c_uint8), ("size", C.c_uint64),
                ("done_cell", C.c_uint64), ("enqueue_ns", C.c_uint64), ("aux", C.c_uint64),
                ("checksum", C.c_uint64), ("scalars", C.c_double * 8), ("views", View * 5),
                ("reserved2", C.c_uint64 * 2)]


class Cfg(C.Structure):
    _fields_ = [("capacity", C.c_uint64), ("table_slots", C.c_uint32), ("num_workers", C.c_uint32),
                ("threads_per_worker", C.c_uint32), ("spin_iterations", C.c_uint32),
                ("backoff_max_exp", C.c_uint32), ("telemetry", C.c_uint32), ("yield_every", C.c_uint64),
                ("trace_capacity", C.c_uint64), ("flags", C.c_uint64), ("reserved", C.c_uint64 * 3)]


class Snapshot(C.Structure):
    _fields_ = [("head", C.c_uint64), ("tail", C.c_uint64), ("processed", C.c_uint64)]


class DevStats(C.Structure):
    _fields_ = [("processed", C.c_uint64), ("failed", C.c_uint64), ("canary_hits", C.c_uint64),
                ("stalls", C.c_uint64), ("torn_reads", C.c_uint64), ("per_op", C.c_uint64 * 256)]


class Tracepoint(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("op_id", C.c_uint64), ("worker", C.c_uint32),
                ("reserved", C.c_uint32), ("enqueue_ns", C.c_uint64), ("dequeue_ns", C.c_uint64),
                ("exec_ns", C.c_uint64), ("version", C.c_uint64)]


class TracePhase(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("enqueue_ns", C.c_uint64), ("ticket_ns", C.c_uint64),
                ("seen_ns", C.c_uint64), ("dequeue_ns", C.c_uint64), ("end_ns", C.c_uint64),
                ("done_ns", C.c_uint64), ("worker", C.c_uint32), ("reserved", C.c_uint32)]


class Instr(C.Structure):
    _fields_ = [("op", C.c_uint8), ("pad", C.c_uint8 * 3), ("k", C.c_int32), ("value", C.c_double)]


class InjectStats(C.Structure):
    _fields_ = [("upload_ns", C.c_uint64), ("epoch_wait_ns", C.c_uint64), ("bank_write_ns", C.c_uint64),
                ("flip_ns", C.c_uint64), ("version", C.c_uint64)]


assert C.sizeof(View) == 48 and C.sizeof(Task) == SLOT_BYTES and C.sizeof(Instr) == 16

# Every symbol include/gpuos_cuda.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "gpuos_abi_version", "gpuos_default_cfg", "gpuos_dev_open", "gpuos_dev_close", "gpuos_dev_alive",
    "gpuos_dev_stop", "gpuos_dev_start", "gpuos_dev_num_workers", "gpuos_dev_sm_count",
    "gpuos_set_yield_every", "gpuos_dev_hold", "gpuos_dev_run_finite", "gpuos_ring_submit_dense", "gpuos_ring_view_get", "gpuos_event_done", "gpuos_jit_compile_object", "gpuos_jit_link_worker",
    "gpuos_dev_load_native", "gpuos_table_install_native", "gpuos_program_upload", "gpuos_dev_clock_offset", "gpuos_buf_alloc", "gpuos_buf_free",
    "gpuos_buf_lookup", "gpuos_buf_copy", "gpuos_buf_fill", "gpuos_buf_prefetch", "gpuos_view_bind", "gpuos_cells_alloc",
    "gpuos_ring_capacity", "gpuos_ring_reserve", "gpuos_ring_publish", "gpuos_ring_peek",
    "gpuos_ring_wait_processed", "gpuos_dev_debug", "gpuos_table_slots", "gpuos_table_version", "gpuos_table_status",
    "gpuos_table_install_builtin", "gpuos_table_install_program", "gpuos_table_kill",
    "gpuos_dev_get_stats", "gpuos_trace_enable", "gpuos_trace_snapshot", "gpuos_trace_phases", "gpuos_launch_task", "gpuos_launch_lean_add",
    "gpuos_stream_create", "gpuos_stream_sync", "gpuos_stream_destroy", "gpuos_dev_kernel_stream",
    "gpuos_event_create", "gpuos_event_record", "gpuos_event_sync", "gpuos_event_elapsed_ms",
    "gpuos_event_destroy", "gpuos_host_alloc", "gpuos_copy_async", "gpuos_jit_compile", "gpuos_free",
    "gpuos_error_name",
]

_lib: Optional[C.CDLL] = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libgpuos_cuda.so; raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libgpuos_cuda.so not built at {path}; run __graft_entry__.build()")
    lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
    P, U64, U32, I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int
    sig = {
        "gpuos_abi_version": ([], I),
        "gpuos_default_cfg": ([C.POINTER(Cfg)], I),
        "gpuos_dev_open": ([I, C.POINTER(Cfg), C.POINTER(P)], I),
        "gpuos_dev_close": ([P], I),
        "gpuos_dev_alive": ([P], I),
        "gpuos_dev_stop": ([P], I),
        "gpuos_dev_start": ([P], I),
        "gpuos_dev_num_workers": ([P, C.POINTER(U32)], I),
        "gpuos_dev_sm_count": ([P, C.POINTER(U32)], I),
        "gpuos_set_yield_every": ([P, U64], I),
        "gpuos_dev_hold": ([P, I], I),
        "gpuos_dev_run_finite": ([P, C.POINTER(C.c_float)], I),
        "gpuos_ring_submit_dense": ([P, P], I),
        "gpuos_ring_view_get": ([P, P], I),
        "gpuos_event_done": ([P, P], I),
        "gpuos_jit_compile_object": ([C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t),
                                      C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t], I),
        "gpuos_jit_link_worker": ([P, P, I, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_uint64),
                                   C.c_char_p, C.c_size_t], I),
        "gpuos_dev_load_native": ([P, P, C.c_size_t, P, P, I, P], I),
        "gpuos_table_install_native": ([P, C.c_uint32, C.c_uint32, P, C.c_uint32, I, I, P], I),
        "gpuos_program_upload": ([P, P, C.c_uint32, I, I, C.POINTER(C.c_uint64)], I),
        "gpuos_dev_clock_offset": ([P, C.POINTER(C.c_int64)], I),
        "gpuos_buf_alloc": ([P, I, U64, C.POINTER(U64), C.POINTER(P)], I),
        "gpuos_buf_free": ([P, U64], I),
        "gpuos_buf_lookup": ([P, U64, C.POINTER(I), C.POINTER(U64), C.POINTER(P)], I),
        "gpuos_buf_copy": ([P, P, P, U64, I], I),
        "gpuos_buf_fill": ([P, P, I, U64], I),
        "gpuos_buf_prefetch": ([P, U64], I),
        "gpuos_view_bind": ([P, U64, I, C.c_int64, I, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                             C.POINTER(View)], I),
        "gpuos_cells_alloc": ([P, U64, C.POINTER(C.POINTER(U64)), C.POINTER(U64)], I),
        "gpuos_ring_capacity": ([P, C.POINTER(U64)], I),
        "gpuos_ring_reserve": ([P, C.POINTER(U64)], I),
        "gpuos_ring_publish": ([P, U64, C.POINTER(Task)], I),
        "gpuos_ring_peek": ([P, C.POINTER(Snapshot)], I),
        "gpuos_ring_wait_processed": ([P, U64], I),
        "gpuos_dev_debug": ([P, C.c_char_p, C.c_size_t], I),
        "gpuos_table_slots": ([P, C.POINTER(U32)], I),
        "gpuos_table_version": ([P, C.POINTER(U64)], I),
        "gpuos_table_status": ([P, U32, C.POINTER(I), C.POINTER(I)], I),
        "gpuos_table_install_builtin": ([P, U32, U32], I),
        "gpuos_table_install_program": ([P, U32, C.POINTER(Instr), U32, I, I, C.POINTER(InjectStats)], I),
        "gpuos_table_kill": ([P, U32], I),
        "gpuos_dev_get_stats": ([P, C.POINTER(DevStats)], I),
        "gpuos_trace_enable": ([P, I], I),
        "gpuos_trace_snapshot": ([P, C.POINTER(Tracepoint), U64, C.POINTER(U64)], I),
        "gpuos_trace_phases": ([P, C.POINTER(TracePhase), U64, C.POINTER(U64)], I),
        "gpuos_launch_task": ([P, C.POINTER(Task), P], I),
        "gpuos_launch_lean_add": ([P, P, P, P, C.c_int64, P], I),
        "gpuos_stream_create": ([P, C.POINTER(P)], I),
        "gpuos_stream_sync": ([P, P], I),
        "gpuos_stream_destroy": ([P, P], I),
        "gpuos_dev_kernel_stream": ([P, C.POINTER(P)], I),
        "gpuos_event_create": ([P, C.POINTER(P)], I),
        "gpuos_event_record": ([P, P, P], I),
        "gpuos_event_sync": ([P, P], I),
        "gpuos_event_elapsed_ms": ([P, P, P, C.POINTER(C.c_float)], I),
        "gpuos_event_destroy": ([P, P], I),
        "gpuos_host_alloc": ([P, U64, C.POINTER(P)], I),
        "gpuos_copy_async": ([P, P, P, U64, I, P], I),
        "gpuos_jit_compile": ([C.c_char_p, C.POINTER(C.c_char_p), I, C.POINTER(P), C.POINTER(C.c_size_t),
                               C.POINTER(U64), C.POINTER(U64), C.c_char_p, C.c_size_t], I),
        "gpuos_free": ([P], None),
        "gpuos_error_name": ([I], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


class GpuosError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        super().__init__(f"{ERRORS[code] if 0 <= code < len(ERRORS) else code}: {what}")


def _ck(rc: int, what: str) -> None:
    if rc != 0:
        raise GpuosError(rc, what)


class Buffer:
    """A device buffer (BufferPool entry, reference tensor.hpp:259-327)."""

    def __init__(self, dev: "Device", id_: int, dtype: int, n: int, ptr: int):
        self.dev, self.id, self.dtype, self.n, self.ptr = dev, id_, dtype, n, ptr

    def write(self, arr: np.ndarray) -> None:
        a = np.ascontiguousarray(arr)
        assert a.nbytes <= self.n * DTYPE_WIDTH[self.dtype]
        _ck(self.dev.lib.gpuos_buf_copy(self.dev.h, self.ptr, a.ctypes.data, a.nbytes, 0), "buf write")

    def read(self, np_dtype) -> np.ndarray:
        out = np.empty(self.n * DTYPE_WIDTH[self.dtype], dtype=np.uint8)
        if out.nbytes:
            _ck(self.dev.lib.gpuos_buf_copy(self.dev.h, out.ctypes.data, self.ptr, out.nbytes, 1), "buf read")
        return out.view(np_dtype)


class Device:
    """One GPU's runtime through the C-ABI: ring, table, buffers, cells."""

    def __init__(self, device: int = 0, capacity: int = 4096, num_workers: int = 0, telemetry: bool = True,
                 table_slots: int = 1024, trace_capacity: int = 65536, install_builtins: bool = True,
                 cells: int = 1 << 16, defer_start: bool = False):
        self.lib = load_library()
        cfg = Cfg()
        self.lib.gpuos_default_cfg(C.byref(cfg))
        cfg.capacity, cfg.num_workers, cfg.telemetry = capacity, num_workers, int(telemetry)
        cfg.table_slots, cfg.trace_capacity = table_slots, trace_capacity
        if defer_start:
            cfg.flags |= CFG_DEFER_START
        h = C.c_void_p()
        _ck(self.lib.gpuos_dev_open(device, C.byref(cfg), C.byref(h)), "dev_open")
        self.h = h
        self._seq = 0
        cptr = C.POINTER(C.c_uint64)()
        daddr = C.c_uint64()
        _ck(self.lib.gpuos_cells_alloc(self.h, cells, C.byref(cptr), C.byref(daddr)), "cells_alloc")
        self.ncells = cells
        self.cells = np.ctypeslib.as_array(cptr, shape=(cells,))
        self.cells_dev = daddr.value
        self._next_cell = 0
        if install_builtins:
            for k in range(14):
                _ck(self.lib.gpuos_table_install_builtin(self.h, k, k), "install builtin")

    # -- lifecycle --
    def close(self) -> None:
        if self.h:
            self.lib.gpuos_dev_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def alive(self) -> bool:
        return bool(self.lib.gpuos_dev_alive(self.h))

    def stop(self) -> None:
        _ck(self.lib.gpuos_dev_stop(self.h), "stop")

    def start(self) -> int:
        return self.lib.gpuos_dev_start(self.h)

    def run_finite(self) -> float:
        """With no resident generation: drain everything published so far with
        one finite worker generation (sentinel behind it); returns its kernel ms."""
        ms = C.c_float()
        _ck(self.lib.gpuos_dev_run_finite(self.h, C.byref(ms)), "run_finite")
        return ms.value

    def hold(self, on: bool) -> None:
        _ck(self.lib.gpuos_dev_hold(self.h, int(on)), "hold")

    # -- buffers / views --
    def alloc(self, dtype: int, n: int) -> Buffer:
        bid, ptr = C.c_uint64(), C.c_void_p()
        _ck(self.lib.gpuos_buf_alloc(self.h, dtype, n, C.byref(bid), C.byref(ptr)), "buf_alloc")
        return Buffer(self, bid.value, dtype, n, ptr.value or 0)

    def free(self, buf: Buffer) -> int:
        return self.lib.gpuos_buf_free(self.h, buf.id)

    def view(self, buf_id: int, dtype: int, shape: Sequence[int], strides: Optional[Sequence[int]] = None,
             offset: int = 0) -> View:
        shape = list(shape)
        if strides is None:
            strides, acc = [0] * len(shape), 1
            for d in range(len(shape) - 1, -1, -1):
                strides[d] = acc
                acc *= shape[d]
        ext = (C.c_int64 * 4)(*shape)
        st = (C.c_int64 * 4)(*strides)
        v = View()
        _ck(self.lib.gpuos_view_bind(self.h, buf_id, dtype, offset, len(shape), ext, st, C.byref(v)), "view_bind")
        return v

    # -- tasks --
    def make_task(self, op_id: int, out: View, inputs: Sequence[View] = (), scalars: Sequence[float] = (),
                  flags: int = 0, cell: bool = True) -> Task:
        t = Task()
        self._seq += 1
        t.seq = self._seq
        t.op_id = op_id
        t.flags = flags
        t.n_inputs = len(inputs)
        t.n_scalars = len(scalars)
        t.views[0] = out
        for i, v in enumerate(inputs):
            t.views[1 + i] = v
        for i, s in enumerate(scalars):
            t.scalars[i] = s
        n = 1
        for d in range(out.rank):
            n *= out.extents[d]
        t.size = n
        if cell:
            idx = self._next_cell % self.ncells
            self._next_cell += 1
            self.cells[idx] = 0
            t.done_cell = self.cells_dev + 8 * idx  # aux stays 0: the task keeps the compact slot format
        return t

    def submit(self, t: Task) -> int:
        pos = C.c_uint64()
        while True:
            rc = self.lib.gpuos_ring_reserve(self.h, C.byref(pos))
            if rc == 0:
                break
            if rc != ERR["QueueFull"]:
                raise GpuosError(rc, "reserve")
            time.sleep(0)
        _ck(self.lib.gpuos_ring_publish(self.h, pos.value, C.byref(t)), "publish")
        return pos.value

    def wait_cell(self, t: Task, timeout: float = 10.0) -> int:
        """Block until the task's completion cell is terminal; returns its ErrorCode."""
        idx = (t.done_cell - self.cells_dev) // 8
        t0 = time.time()
        while True:
            w = int(self.cells[idx])
            if w & 0xFF:
                return (w >> 8) & 0xFF
            if time.time() - t0 > timeout:
                raise TimeoutError(f"task seq={t.seq} op={t.op_id} not completed: {self.debug()}")

    def run(self, op_id: int, out: View, inputs: Sequence[View] = (), scalars: Sequence[float] = (),
            flags: int = 0) -> int:
        t = self.make_task(op_id, out, inputs, scalars, flags)
        self.submit(t)
        return self.wait_cell(t)

    def launch(self, t: Task, stream: Optional[int] = None) -> int:
        """Conventional path: one cudaLaunchKernel of the same task body."""
        return self.lib.gpuos_launch_task(self.h, C.byref(t), stream)

    def run_inline(self, op_id: int, out: View, inputs: Sequence[View] = (), scalars: Sequence[float] = (),
                   flags: int = 0) -> int:
        t = self.make_task(op_id, out, inputs, scalars, flags)
        rc = self.launch(t)
        if rc != 0:
            return rc
        _ck(self.lib.gpuos_stream_sync(self.h, None), "stream_sync")
        return self.wait_cell(t)

    def wait_processed(self, count: int) -> None:
        _ck(self.lib.gpuos_ring_wait_processed(self.h, count), "wait_processed")

    def debug(self) -> str:
        buf = C.create_string_buffer(4096)
        self.lib.gpuos_dev_debug(self.h, buf, 4096)
        return buf.value.decode()

    def peek(self) -> Snapshot:
        s = Snapshot()
        _ck(self.lib.gpuos_ring_peek(self.h, C.byref(s)), "peek")
        return s

    # -- table --
    def version(self) -> int:
        v = C.c_uint64()
        _ck(self.lib.gpuos_table_version(self.h, C.byref(v)), "version")
        return v.value

    def status(self, op_id: int):
        s, k = C.c_int(), C.c_int()
        rc = self.lib.gpuos_table_status(self.h, op_id, C.byref(s), C.byref(k))
        return rc, s.value, k.value

    def install_builtin(self, op_id: int, kind: int) -> int:
        return self.lib.gpuos_table_install_builtin(self.h, op_id, kind)

    def install_program(self, op_id: int, code: Sequence[tuple], arity: int, dtype: int):
        arr = (Instr * len(code))()
        for i, ins in enumerate(code):
            arr[i].op = ins[0]
            arr[i].k = ins[1] if len(ins) > 1 else 0
            arr[i].value = ins[2] if len(ins) > 2 else 0.0
        st = InjectStats()
        rc = self.lib.gpuos_table_install_program(self.h, op_id, arr, len(code), arity, dtype, C.byref(st))
        return rc, st

    def kill(self, op_id: int) -> int:
        return self.lib.gpuos_table_kill(self.h, op_id)

    def stats(self) -> DevStats:
        s = DevStats()
        _ck(self.lib.gpuos_dev_get_stats(self.h, C.byref(s)), "stats")
        return s

    def phases(self, cap: int = 65536):
        arr = (TracePhase * cap)()
        n = C.c_uint64()
        _ck(self.lib.gpuos_trace_phases(self.h, arr, cap, C.byref(n)), "phases")
        return [arr[i] for i in range(n.value)]

    def trace(self, cap: int = 65536):
        arr = (Tracepoint * cap)()
        n = C.c_uint64()
        _ck(self.lib.gpuos_trace_snapshot(self.h, arr, cap, C.byref(n)), "trace")
        return [arr[i] for i in range(n.value)]
