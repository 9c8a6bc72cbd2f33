"""Run a parity case through the oracle, the reference, or the B200 runtime
(C-ABI) and compare results under the case's tolerance rule."""
from __future__ import annotations

import math
from typing import List, Optional, Tuple

import numpy as np

import oracle_lib as ol
from cases import BF16, F16, F32, F64, I32, Case, Operand

ERRORS = ["Ok", "IncompatibleShapes", "OutOfBounds", "InvalidBuffer", "ZeroCapacity", "QueueFull", "ZeroSlots",
          "OutOfRange", "NotInstalled", "OperatorKilled", "TableFull", "SyntaxError", "UnknownIdentifier",
          "ArityError", "VerifyError", "EmptyAxis", "DTypeMismatch", "ShapeMismatch", "TooLarge", "OddDim",
          "CacheFull", "AlreadyStarted", "RuntimeStopped", "IoError", "Internal"]


def storage(op: Operand) -> np.ndarray:
    return ol.encode(op.values, op.dtype)


def host_tensor(op: Operand) -> ol.HostTensor:
    return ol.HostTensor(storage(op), op.dtype, op.shape, op.strides, op.offset)


def _run_host(case: Case, runner) -> Tuple[int, List[np.ndarray]]:
    ins = [host_tensor(o) for o in case.inputs]
    out = host_tensor(case.out)
    rc = runner(case.op, out, ins, case.scalars, case.uncapped)
    bufs = [out.buf] + ([ins[2].buf] if case.op == "kv_append" else [])
    return rc, bufs


def oracle_run(case: Case):
    return _run_host(case, ol.run_oracle)


def reference_run(case: Case):
    return _run_host(case, ol.run_reference)


def device_run(dev, case: Case, inline: bool = False):
    """The same case through the B200 runtime: buffers in HBM, one task on
    the ring (or one cudaLaunchKernel when inline)."""
    from paper_2604_17861_b200 import abi
    bufs = []
    views = []
    for o in case.inputs + [case.out]:
        data = storage(o)
        b = dev.alloc(o.dtype, data.size)
        b.write(data)
        bufs.append(b)
        views.append(dev.view(b.id, o.dtype, o.shape, o.strides, o.offset))
    out_view = views[-1]
    flags = abi.FLAG_UNCAPPED if case.uncapped else 0
    op_id = abi.OP[case.op]
    if inline:
        rc = dev.run_inline(op_id, out_view, views[:-1], case.scalars, flags)
    else:
        rc = dev.run(op_id, out_view, views[:-1], case.scalars, flags)
    np_t = ol.NP[case.out.dtype]
    outs = [bufs[-1].read(np_t)[: storage(case.out).size]]
    if case.op == "kv_append":
        outs.append(bufs[2].read(ol.NP[case.inputs[2].dtype])[: storage(case.inputs[2]).size])
    for b in bufs:
        dev.free(b)
    return rc, outs


def logical(op: Operand) -> np.ndarray:
    """The view's logical values (after narrowing to its dtype), shape op.shape."""
    vals = ol.decode(storage(op), op.dtype)
    idx = np.full(op.shape, op.offset, dtype=np.int64) if op.shape else np.array(op.offset)
    for d, (e, s) in enumerate(zip(op.shape, op.strides)):
        sh = [1] * len(op.shape)
        sh[d] = e
        idx = idx + (np.arange(e, dtype=np.int64) * s).reshape(sh)
    return vals[idx]


def _ulp_dist(a: np.ndarray, b: np.ndarray, dtype: int) -> np.ndarray:
    """|ordered-integer distance| between encodings (NaN handled by callers)."""
    if dtype == F32:
        ia, ib = a.view(np.int32).astype(np.int64), b.view(np.int32).astype(np.int64)
        sign = np.int64(1 << 31)
    elif dtype == F64:
        ia, ib = a.view(np.int64).astype(object), b.view(np.int64).astype(object)
        return np.array([abs(int(x) - int(y)) for x, y in zip(ia, ib)], dtype=object)
    else:
        ia, ib = a.astype(np.int64), b.astype(np.int64)
        sign = np.int64(1 << 15)
    fa = np.where(ia & sign, sign - ia, ia) if dtype != F32 else np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    fb = np.where(ib & sign, sign - ib, ib) if dtype != F32 else np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    return np.abs(fa - fb)


def compare(case: Case, got: np.ndarray, want: np.ndarray, dtype: int) -> Tuple[bool, str, float]:
    """Returns (ok, message, bit-exact fraction)."""
    if got.size != want.size:
        return False, f"size {got.size} vs {want.size}", 0.0
    if got.size == 0:
        return True, "", 1.0
    g = ol.decode(got, dtype)
    w = ol.decode(want, dtype)
    both_nan = np.isnan(g) & np.isnan(w)
    same_bits = (got.view(np.uint8).reshape(got.size, -1) == want.view(np.uint8).reshape(want.size, -1)).all(1)
    exact = same_bits | both_nan
    frac = float(exact.mean())
    rule = case.rule
    if rule == "exact":
        # bit-exact; NaN payloads may differ (narrowing canonicalises them)
        if not exact.all():
            i = int(np.argmax(~exact))
            return False, f"not exact at {i}: got {g[i]!r} want {w[i]!r}", frac
        return True, "", frac
    if rule == "ulp1":
        bad = ~exact & (np.isnan(g) | np.isnan(w))
        if bad.any():
            return False, "NaN mismatch", frac
        d = _ulp_dist(got, want, dtype)
        if (np.array(d, dtype=np.float64) > 1).any():
            i = int(np.argmax(np.array(d, dtype=np.float64)))
            return False, f"{d[i]} ulp at {i}: got {g[i]!r} want {w[i]!r}", frac
        return True, "", frac
    if rule == "gemm32":
        # tensor-core GEMM (bf16/f16 in, fp32 accumulate, one rounding to the
        # output dtype) vs the reference's fp64 ascending-k sum: within one
        # output ulp plus the fp32 accumulation bound k * 2^-23 * sum|a||b|
        a, b = logical(case.inputs[0]), logical(case.inputs[1])
        k = a.shape[1]
        acc_bound = (k * 2.0 ** -23) * (np.abs(a) @ np.abs(b)).ravel()
        wf = w.astype(np.float32)
        ulp = np.spacing(np.abs(wf)).astype(np.float64) * (2.0 ** 16 if dtype == BF16 else 2.0 ** 13)
        if dtype == F16:
            ulp = np.spacing(np.abs(w.astype(np.float16))).astype(np.float64)
        err = np.abs(g - w)
        lim = ulp + acc_bound
        if (err > lim).any() or np.isnan(err).any():
            i = int(np.argmax(err - lim))
            return False, f"err {err[i]:.3e} > bound {lim[i]:.3e} at {i}: got {g[i]!r} want {w[i]!r}", frac
        return True, "", frac
    tol = float(rule.split(":")[1])
    scale = np.maximum(1.0, np.abs(w))
    err = np.where(both_nan, 0.0, np.abs(g - w))
    err = np.where(np.isnan(err), np.inf, err)
    if (err > tol * scale).any():
        i = int(np.argmax(err / scale))
        return False, f"rel err {err[i] / scale[i]:.3e} > {tol} at {i}: got {g[i]!r} want {w[i]!r}", frac
    return True, "", frac
