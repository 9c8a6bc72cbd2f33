"""Seeded parity cases shared by the CPU oracle-vs-reference tests and the GPU
parity tests.  Each case describes operand buffers, strided views into them
(contiguous, stride-2, transposed, negative-stride, broadcast, rank-0), the
op, its scalars, and the tolerance rule SURVEY.md §8(a) assigns to it.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

F32, F64, I32, F16, BF16 = 0, 1, 2, 3, 4
FLOAT_DTYPES = (F32, F64, F16, BF16)
ALL_DTYPES = (F32, F64, I32, F16, BF16)


@dataclasses.dataclass
class Operand:
    values: np.ndarray            # doubles for the whole buffer (pre-narrowing)
    dtype: int
    shape: List[int]
    strides: List[int]
    offset: int = 0


@dataclasses.dataclass
class Case:
    name: str
    op: str
    dtype: int
    inputs: List[Operand]
    out: Operand
    scalars: List[float]
    rule: str                      # "exact" | "ulp1" | "rel:<tol>"
    uncapped: bool = False
    extra: Optional[Operand] = None


def contiguous(shape: Sequence[int]) -> List[int]:
    st, acc = [0] * len(shape), 1
    for d in range(len(shape) - 1, -1, -1):
        st[d] = acc
        acc *= shape[d]
    return st


def numel(shape: Sequence[int]) -> int:
    n = 1
    for e in shape:
        n *= e
    return n


def rand_vals(rng, n, dtype, lo=-4.0, hi=4.0, op="add"):
    if dtype == I32:
        if op == "mul":
            return rng.integers(-(2 ** 15), 2 ** 15, n).astype(np.float64)
        return rng.integers(-(2 ** 30), 2 ** 30, n).astype(np.float64)
    return rng.uniform(lo, hi, n)


def layout(rng, shape, dtype, kind, op="add", lo=-4.0, hi=4.0) -> Operand:
    """An operand of logical `shape` laid out as `kind` in a fresh buffer."""
    n = numel(shape)
    if kind == "contig" or len(shape) == 0:
        return Operand(rand_vals(rng, max(n, 1), dtype, lo, hi, op), dtype, list(shape), contiguous(shape))
    if kind == "stride2":
        st = [s * 2 for s in contiguous(shape)]
        return Operand(rand_vals(rng, max(2 * n, 1), dtype, lo, hi, op), dtype, list(shape), st)
    if kind == "transposed" and len(shape) == 2:
        r, c = shape
        return Operand(rand_vals(rng, max(n, 1), dtype, lo, hi, op), dtype, list(shape), [1, r])
    if kind == "negative":
        st = [-s for s in contiguous(shape)]
        return Operand(rand_vals(rng, max(n, 1), dtype, lo, hi, op), dtype, list(shape), st, offset=max(n - 1, 0))
    return Operand(rand_vals(rng, max(n, 1), dtype, lo, hi, op), dtype, list(shape), contiguous(shape))


def out_operand(shape, dtype) -> Operand:
    return Operand(np.zeros(max(numel(shape), 1)), dtype, list(shape), contiguous(shape))


def elementwise_cases(seed=7, dtypes=ALL_DTYPES) -> List[Case]:
    rng = np.random.default_rng(seed)
    cases = []
    shapes = [[4096], [64, 64], [3, 5, 7], [2, 3, 4, 5], [1000]]
    for op in ("add", "mul", "relu", "gelu"):
        for dt in dtypes:
            if op == "gelu" and dt == I32:
                continue
            rule = "exact" if op != "gelu" else ("rel:1e-6" if dt == F32 else "rel:1e-12" if dt == F64 else "ulp1")
            for si, shape in enumerate(shapes):
                for kind in ("contig", "stride2", "transposed", "negative"):
                    if kind == "transposed" and len(shape) != 2:
                        continue
                    arity = 2 if op in ("add", "mul") else 1
                    ins = [layout(rng, shape, dt, kind if i == 0 else "contig", op) for i in range(arity)]
                    cases.append(Case(f"{op}-{dt}-{si}-{kind}", op, dt, ins, out_operand(shape, dt), [], rule))
            # broadcast: (1,C) against (R,C); rank-0 scalar against (n)
            if op in ("add", "mul"):
                a = layout(rng, [48, 33], dt, "contig", op)
                b = layout(rng, [1, 33], dt, "contig", op)
                cases.append(Case(f"{op}-{dt}-bcast-row", op, dt, [a, b], out_operand([48, 33], dt), [], rule))
                a = layout(rng, [513], dt, "contig", op)
                s = layout(rng, [], dt, "contig", op)
                cases.append(Case(f"{op}-{dt}-bcast-scalar", op, dt, [a, s], out_operand([513], dt), [], rule))
                a = layout(rng, [7, 1], dt, "contig", op)
                b = layout(rng, [1, 9], dt, "contig", op)
                cases.append(Case(f"{op}-{dt}-bcast-outer", op, dt, [a, b], out_operand([7, 9], dt), [], rule))
    # special values: -0.0 and NaN through relu
    for dt in (F32, F64, F16, BF16):
        vals = np.array([-0.0, 0.0, np.nan, -np.nan, -1.5, 2.5, -np.inf, np.inf] * 8)
        ins = [Operand(vals, dt, [64], [1])]
        cases.append(Case(f"relu-{dt}-special", "relu", dt, ins, out_operand([64], dt), [], "exact"))
    # empty output
    cases.append(Case("add-empty", "add", F32, [Operand(np.zeros(1), F32, [0, 4], [4, 1]),
                                                 Operand(np.zeros(1), F32, [0, 4], [4, 1])],
                      out_operand([0, 4], F32), [], "exact"))
    return cases


def row_cases(seed=11, dtypes=ALL_DTYPES) -> List[Case]:
    rng = np.random.default_rng(seed)
    cases = []
    for op in ("reduce_sum", "reduce_max", "reduce_min"):
        for dt in dtypes:
            # f64 sums: tree vs sequential reassociation, close_tol(1e-12) as the
            # reference tests use (test_ops.cpp:301); f32/f16/bf16: <= 1 ulp
            rule = "exact" if (op != "reduce_sum" or dt == I32) else ("rel:1e-12" if dt == F64 else "ulp1")
            for shape in ([37, 129], [5, 4096], [3, 4, 65], [1500], [2, 2000]):
                for kind in ("contig", "stride2", "transposed"):
                    if kind == "transposed" and len(shape) != 2:
                        continue
                    inp = layout(rng, shape, dt, kind)
                    cases.append(Case(f"{op}-{dt}-{shape}-{kind}", op, dt, [inp], out_operand(shape[:-1], dt), [], rule))
            # ties / NaN first / -0 vs +0 for max/min first-wins (ops.hpp:334-338)
            if op != "reduce_sum" and dt != I32:
                vals = np.array([[np.nan, 1.0, 2.0, 2.0], [-0.0, 0.0, -0.0, 0.0], [1.0, np.nan, 3.0, 3.0],
                                 [0.0, -0.0, -1.0, 5.0]]).ravel()
                cases.append(Case(f"{op}-{dt}-special", op, dt, [Operand(vals, dt, [4, 4], [4, 1])],
                                  out_operand([4], dt), [], "exact"))
        cases.append(Case(f"{op}-empty-axis", op, F32, [Operand(np.zeros(1), F32, [4, 0], [0, 1])],
                          out_operand([4], F32), [], "exact"))
    for dt in (F32, F64, F16, BF16):
        rule = "rel:1e-6" if dt == F32 else "rel:1e-12" if dt == F64 else "ulp1"
        for shape in ([16, 128], [3, 1000], [2, 3, 64], [1, 3000]):
            inp = layout(rng, shape, dt, "contig", lo=-8, hi=8)
            cases.append(Case(f"softmax-{dt}-{shape}", "softmax", dt, [inp], out_operand(shape, dt), [], rule))
        inp = layout(rng, [32, 48], dt, "transposed", lo=-8, hi=8)
        cases.append(Case(f"softmax-{dt}-transposed", "softmax", dt, [inp], out_operand([32, 48], dt), [], rule))
        rule_ln = "rel:1e-5" if dt == F32 else "rel:1e-12" if dt == F64 else "ulp1"
        for shape in ([8, 96], [2, 3, 1500]):
            c = shape[-1]
            x = layout(rng, shape, dt, "contig")
            g = layout(rng, [c], dt, "contig", lo=0.5, hi=2.0)
            b = layout(rng, [c], dt, "contig", lo=-1, hi=1)
            cases.append(Case(f"layernorm-{dt}-{shape}", "layernorm", dt, [x, g, b], out_operand(shape, dt), [1e-5],
                              rule_ln))
        x = layout(rng, [6, 64], dt, "contig")
        g = layout(rng, [], dt, "contig", lo=0.5, hi=2.0)
        b = layout(rng, [1], dt, "contig")
        cases.append(Case(f"layernorm-{dt}-bcast-gamma", "layernorm", dt, [x, g, b], out_operand([6, 64], dt), [],
                          rule_ln))
    return cases


def linalg_cases(seed=13, dtypes=ALL_DTYPES) -> List[Case]:
    rng = np.random.default_rng(seed)
    cases = []
    for dt in dtypes:
        lo, hi = (-1.0, 1.0)
        for (m, k, n) in ((128, 64, 128), (128, 128, 64), (37, 19, 53), (256, 256, 256), (1, 70, 3)):
            a = layout(rng, [m, k], dt, "contig", "mul" if dt == I32 else "add", lo, hi)
            b = layout(rng, [k, n], dt, "transposed" if n == k else "contig", "mul" if dt == I32 else "add", lo, hi)
            # f16/bf16 run on the tensor cores: fp32 accumulation (bound in parity.compare)
            rule = "gemm32" if dt in (F16, BF16) else "exact"
            cases.append(Case(f"matmul-{dt}-{m}x{k}x{n}", "matmul_small", dt, [a, b], out_operand([m, n], dt), [], rule))
        a = layout(rng, [16, 257], dt, "contig", "mul", lo, hi)
        b = layout(rng, [257, 8], dt, "contig", "mul", lo, hi)
        cases.append(Case(f"matmul-{dt}-toolarge", "matmul_small", dt, [a, b], out_operand([16, 8], dt), [], "exact"))
        v = layout(rng, [96], dt, "contig", "mul", lo, hi)
        mt = layout(rng, [96, 80], dt, "stride2", "mul", lo, hi)
        cases.append(Case(f"vecmat-{dt}", "vecmat", dt, [v, mt], out_operand([80], dt), [], "exact"))
        v = layout(rng, [24], dt, "contig", "mul", lo, hi)
        mt = layout(rng, [24, 16], dt, "contig", "mul", lo, hi)
        cases.append(Case(f"vecmat-{dt}-small", "vecmat", dt, [v, mt], out_operand([16], dt), [], "exact"))
        cases.append(Case(f"vecmat-{dt}-small2", "vecmat", dt, [v, mt], out_operand([16], dt), [], "exact"))
        if dt == I32:
            continue
        rule = "rel:1e-6" if dt == F32 else "rel:1e-12" if dt == F64 else "ulp1"
        for (h, t, d) in ((4, 128, 64), (2, 1, 16), (3, 300, 64), (1, 2048, 8)):
            q = layout(rng, [h, d], dt, "contig", lo=-1, hi=1)
            kk = layout(rng, [h, t, d], dt, "contig", lo=-1, hi=1)
            vv = layout(rng, [h, t, d], dt, "contig", lo=-1, hi=1)
            cases.append(Case(f"sdpa-{dt}-{h}x{t}x{d}", "sdpa", dt, [q, kk, vv], out_operand([h, d], dt), [], rule))
        x = layout(rng, [6, 64], dt, "contig")
        pos = Operand(np.arange(6, dtype=np.float64) * 3.0, I32, [6], [1])
        cases.append(Case(f"rope-{dt}-i32pos", "rope", dt, [x, pos], out_operand([6, 64], dt), [], rule))
        pos2 = Operand(np.arange(5, dtype=np.float64) * 1.25, dt, [5], [1])
        x2 = layout(rng, [5, 10], dt, "contig")
        cases.append(Case(f"rope-{dt}-base", "rope", dt, [x2, pos2], out_operand([5, 10], dt), [500.0], rule))
        x3 = layout(rng, [2, 7], dt, "contig")
        cases.append(Case(f"rope-{dt}-odd", "rope", dt, [x3, Operand(np.zeros(2), dt, [2], [1])],
                          out_operand([2, 7], dt), [], rule))
    # kv_append: k_cache is the output operand; v_cache an input (ops.hpp:578-589)
    for dt in ALL_DTYPES:
        h, cap, d = 2, 5, 8
        nk = layout(rng, [h, d], dt, "contig")
        nv = layout(rng, [h, d], dt, "contig")
        vc = Operand(np.zeros(h * cap * d), dt, [h, cap, d], contiguous([h, cap, d]))
        kc = Operand(np.zeros(h * cap * d), dt, [h, cap, d], contiguous([h, cap, d]))
        for cur in (0.0, 3.0, 5.0, -1.0):
            cases.append(Case(f"kv_append-{dt}-{cur}", "kv_append", dt, [nk, nv, vc], kc, [cur], "exact"))
    return cases
