"""ctypes access to the test-only oracle (oracle/liboracle.so) and to the
reference's own kernels (oracle/_ref/libref.so, built from /root/reference).

Test infrastructure: only tests/ and __graft_entry__.smoke() import this, and
only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref.so")

F32, F64, I32, F16, BF16 = 0, 1, 2, 3, 4
NP = {F32: np.float32, F64: np.float64, I32: np.int32, F16: np.uint16, BF16: np.uint16}
OPS = dict(add=0, mul=1, relu=2, gelu=3, softmax=4, layernorm=5, reduce_sum=6, reduce_max=7, reduce_min=8,
           matmul_small=9, vecmat=10, sdpa=11, rope=12, kv_append=13)


class OrcView(C.Structure):
    _fields_ = [("base", C.c_void_p), ("offset", C.c_int64), ("rank", C.c_int32), ("dtype", C.c_int32),
                ("shape", C.c_int64 * 8), ("strides", C.c_int64 * 8), ("buf_dtype", C.c_int32),
                ("pad", C.c_int32)]


class OrcInstr(C.Structure):
    _fields_ = [("op", C.c_int32), ("k", C.c_int32), ("value", C.c_double)]


class RefTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("buf_len", C.c_int64), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("offset", C.c_int64), ("shape", C.c_int64 * 8), ("strides", C.c_int64 * 8)]


_orc: Optional[C.CDLL] = None
_ref: Optional[C.CDLL] = None


def oracle() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError("oracle/liboracle.so not built (make -C oracle)")
        lib = C.CDLL(ORACLE_SO)
        V = C.POINTER(OrcView)
        lib.orc_elementwise.argtypes = [C.c_int, V, V, C.c_int]
        lib.orc_softmax.argtypes = [V, V]
        lib.orc_layernorm.argtypes = [V, V, V, V, C.c_double, C.c_int]
        lib.orc_reduce.argtypes = [C.c_int, V, V]
        lib.orc_matmul.argtypes = [V, V, V, C.c_int64]
        lib.orc_vecmat.argtypes = [V, V, V, C.c_int64]
        lib.orc_sdpa.argtypes = [V, V, V, V, C.c_double, C.c_int]
        lib.orc_rope.argtypes = [V, V, V, C.c_double, C.c_int]
        lib.orc_kv_append.argtypes = [V, V, V, V, C.c_double]
        lib.orc_program.argtypes = [C.POINTER(OrcInstr), C.c_int, C.c_int, C.c_int, V, V, C.c_int]
        lib.orc_f16_bits.argtypes = [C.c_double]
        lib.orc_f16_bits.restype = C.c_uint16
        lib.orc_bf16_bits.argtypes = [C.c_double]
        lib.orc_bf16_bits.restype = C.c_uint16
        lib.orc_f16_value.argtypes = [C.c_uint16]
        lib.orc_f16_value.restype = C.c_double
        lib.orc_bf16_value.argtypes = [C.c_uint16]
        lib.orc_bf16_value.restype = C.c_double
        lib.orc_narrow.argtypes = [C.c_int, C.c_double]
        lib.orc_narrow.restype = C.c_double
        lib.orc_narrow_i32.argtypes = [C.c_double]
        lib.orc_narrow_i32.restype = C.c_int32
        lib.orc_broadcast_shapes.argtypes = [C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int64), C.c_int,
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        _orc = lib
    return _orc


def reference() -> Optional[C.CDLL]:
    """The reference kernels, or None when oracle/_ref was not built."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        lib = C.CDLL(REF_SO)
        T = C.POINTER(RefTensor)
        lib.ref_run_builtin.argtypes = [C.c_int, C.c_int, T, T, C.POINTER(C.c_double), C.c_int, C.c_int64]
        lib.ref_run_template.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, T, T]
        lib.ref_compile_template.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.c_int, C.c_int,
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                             C.c_int, C.POINTER(C.c_int)]
        _ref = lib
    return _ref


class HostTensor:
    """A host buffer plus a strided view of it (the oracle's operand)."""

    def __init__(self, buf: np.ndarray, dtype: int, shape: Sequence[int], strides: Optional[Sequence[int]] = None,
                 offset: int = 0, buf_dtype: Optional[int] = None):
        self.buf = np.ascontiguousarray(buf)
        self.dtype = dtype
        self.shape = list(shape)
        if strides is None:
            strides, acc = [0] * len(self.shape), 1
            for d in range(len(self.shape) - 1, -1, -1):
                strides[d] = acc
                acc *= self.shape[d]
        self.strides = list(strides)
        self.offset = offset
        self.buf_dtype = dtype if buf_dtype is None else buf_dtype

    def copy(self) -> "HostTensor":
        return HostTensor(self.buf.copy(), self.dtype, self.shape, self.strides, self.offset, self.buf_dtype)

    def orc(self) -> OrcView:
        v = OrcView()
        v.base = self.buf.ctypes.data
        v.offset = self.offset
        v.rank = len(self.shape)
        v.dtype = self.dtype
        for i, (e, s) in enumerate(zip(self.shape, self.strides)):
            v.shape[i] = e
            v.strides[i] = s
        v.buf_dtype = self.buf_dtype
        return v

    def ref(self) -> RefTensor:
        t = RefTensor()
        t.data = self.buf.ctypes.data
        t.buf_len = self.buf.size
        t.dtype = self.dtype
        t.rank = len(self.shape)
        t.offset = self.offset
        for i, (e, s) in enumerate(zip(self.shape, self.strides)):
            t.shape[i] = e
            t.strides[i] = s
        return t


def run_oracle(op: str, out: HostTensor, inputs: Sequence[HostTensor], scalars: Sequence[float] = (),
               uncapped: bool = False) -> int:
    """Run one builtin through the oracle; writes into out.buf (and kv caches)."""
    lib = oracle()
    ov = out.orc()
    ivs = [t.orc() for t in inputs]
    arr = (OrcView * max(1, len(ivs)))(*ivs)
    has = len(scalars) > 0
    s0 = float(scalars[0]) if has else 0.0
    if op in ("add", "mul", "relu", "gelu"):
        return lib.orc_elementwise(OPS[op], C.byref(ov), arr, len(ivs))
    if len(ivs) == 0:
        return 13
    if op == "softmax":
        return lib.orc_softmax(C.byref(ov), C.byref(arr[0])) if len(ivs) == 1 else 13
    if op == "layernorm":
        return lib.orc_layernorm(C.byref(ov), C.byref(arr[0]), C.byref(arr[1]), C.byref(arr[2]), s0, int(has)) \
            if len(ivs) == 3 else 13
    if op.startswith("reduce_"):
        mode = {"reduce_sum": 0, "reduce_max": 1, "reduce_min": 2}[op]
        return lib.orc_reduce(mode, C.byref(ov), C.byref(arr[0])) if len(ivs) == 1 else 13
    if op == "matmul_small":
        return lib.orc_matmul(C.byref(ov), C.byref(arr[0]), C.byref(arr[1]), 0 if uncapped else 256) \
            if len(ivs) == 2 else 13
    if op == "vecmat":
        return lib.orc_vecmat(C.byref(ov), C.byref(arr[0]), C.byref(arr[1]), 0 if uncapped else 256) \
            if len(ivs) == 2 else 13
    if op == "sdpa":
        return lib.orc_sdpa(C.byref(ov), C.byref(arr[0]), C.byref(arr[1]), C.byref(arr[2]), s0, int(has)) \
            if len(ivs) == 3 else 13
    if op == "rope":
        return lib.orc_rope(C.byref(ov), C.byref(arr[0]), C.byref(arr[1]), s0, int(has)) if len(ivs) == 2 else 13
    if op == "kv_append":
        # descriptor form: inputs {new_k, new_v, v_cache}, output k_cache (ops.hpp:578-589)
        if len(ivs) != 3:
            return 13
        if not has:
            return 13
        rc = lib.orc_kv_append(C.byref(ov), C.byref(arr[2]), C.byref(arr[0]), C.byref(arr[1]), s0)
        return rc
    raise ValueError(op)


def run_reference(op: str, out: HostTensor, inputs: Sequence[HostTensor], scalars: Sequence[float] = (),
                  uncapped: bool = False) -> int:
    lib = reference()
    assert lib is not None
    ov = out.ref()
    ivs = (RefTensor * max(1, len(inputs)))(*[t.ref() for t in inputs])
    sc = (C.c_double * max(1, len(scalars)))(*scalars)
    rc = lib.ref_run_builtin(OPS[op], len(inputs), ivs, C.byref(ov), sc, len(scalars), 0 if uncapped else 256)
    return rc


def program(code: Sequence[tuple]):
    arr = (OrcInstr * len(code))()
    for i, ins in enumerate(code):
        arr[i].op = ins[0]
        arr[i].k = ins[1] if len(ins) > 1 else 0
        arr[i].value = ins[2] if len(ins) > 2 else 0.0
    return arr


def run_program(code: Sequence[tuple], arity: int, dtype: int, out: HostTensor, inputs: Sequence[HostTensor]) -> int:
    arr = program(code)
    ivs = (OrcView * max(1, len(inputs)))(*[t.orc() for t in inputs])
    ov = out.orc()
    return oracle().orc_program(arr, len(code), arity, dtype, C.byref(ov), ivs, len(inputs))


def compile_template_ref(source: str, params: Sequence[float], arity: int):
    """Lower + verify a template through the reference; returns [(op,k,value)], max_stack."""
    lib = reference()
    assert lib is not None
    cap = 512
    ops, ks, vals = (C.c_int32 * cap)(), (C.c_int32 * cap)(), (C.c_double * cap)()
    ms = C.c_int()
    p = (C.c_double * 8)(*(list(params) + [0.0] * (8 - len(params))))
    n = lib.ref_compile_template(source.encode(), p, 8, arity, ops, ks, vals, cap, C.byref(ms))
    if n < 0:
        return None, -n
    return [(ops[i], ks[i], vals[i]) for i in range(n)], ms.value


# ---- value generation / encoding helpers shared by the tests ----

def encode(vals: np.ndarray, dtype: int) -> np.ndarray:
    """Store doubles into a buffer of `dtype` with the oracle's narrowing."""
    lib = oracle()
    vals = np.asarray(vals, dtype=np.float64).ravel()
    if dtype == F32:
        return vals.astype(np.float32)
    if dtype == F64:
        return vals.copy()
    if dtype == I32:
        return np.array([lib.orc_narrow_i32(float(v)) for v in vals], dtype=np.int32)
    fn = lib.orc_f16_bits if dtype == F16 else lib.orc_bf16_bits
    return np.array([fn(float(v)) for v in vals], dtype=np.uint16)


def decode(buf: np.ndarray, dtype: int) -> np.ndarray:
    lib = oracle()
    if dtype in (F32, F64, I32):
        return buf.astype(np.float64)
    fn = lib.orc_f16_value if dtype == F16 else lib.orc_bf16_value
    return np.array([fn(int(b)) for b in buf], dtype=np.float64)
