"""Generate golden fixtures from the reference itself (run in the container
where /root/reference exists; the fixtures travel, the reference does not).

  python tests/golden/make_golden.py

programs.json : the nine shipped templates lowered + verified by the reference
                (bytecode.hpp:135-201) with params (0.75, 2.5)
builtins.json : small seeded cases run through the reference kernels
                (oracle/_ref/libref.so): inputs, error code, outputs (hex bytes)
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

import oracle_lib as ol  # noqa: E402
from cases import F32, F64, I32, elementwise_cases, linalg_cases, row_cases  # noqa: E402
from parity import reference_run, storage  # noqa: E402

TEMPLATES = [("scale_add", "in0 * $p0 + $p1", 1), ("clamp", "min(max(in0, $p0), $p1)", 1),
             ("sigmoid", "1 / (1 + exp(-in0))", 1), ("silu", "in0 / (1 + exp(-in0))", 1),
             ("leaky_relu", "max(in0, 0) + $p0 * min(in0, 0)", 1), ("tanh_gate", "tanh(in0) * in1", 2),
             ("abs_diff", "abs(in0 - in1)", 2), ("fma", "in0 * in1 + in2", 3),
             ("inv_sqrt_scale", "in0 / sqrt($p0 + in0 * in0)", 1)]


def main():
    assert ol.reference() is not None, "build oracle/_ref first (make -C oracle)"
    progs = {}
    for name, src, arity in TEMPLATES:
        code, ms = ol.compile_template_ref(src, [0.75, 2.5], arity)
        progs[name] = {"source": src, "arity": arity, "params": [0.75, 2.5], "code": code, "max_stack": ms}
    with open(os.path.join(HERE, "programs.json"), "w") as f:
        json.dump(progs, f, indent=1)

    cases = [c for c in elementwise_cases(dtypes=(F32, F64, I32)) + row_cases(dtypes=(F32, F64, I32)) +
             linalg_cases(dtypes=(F32, F64, I32))
             if all(o.dtype in (F32, F64, I32) for o in c.inputs) and c.out.values.size <= 1100 and
             sum(o.values.size for o in c.inputs) <= 4200]
    out = []
    for c in cases[::2]:
        rc, bufs = reference_run(c)
        out.append({
            "name": c.name, "op": c.op, "dtype": c.dtype, "scalars": c.scalars, "rule": c.rule,
            "inputs": [{"dtype": o.dtype, "shape": o.shape, "strides": o.strides, "offset": o.offset,
                        "data": storage(o).tobytes().hex()} for o in c.inputs],
            "out": {"dtype": c.out.dtype, "shape": c.out.shape, "strides": c.out.strides, "offset": c.out.offset,
                    "size": int(storage(c.out).size)},
            "code": rc, "results": [b.tobytes().hex() for b in bufs],
        })
    with open(os.path.join(HERE, "builtins.json"), "w") as f:
        json.dump(out, f)
    print(f"wrote {len(progs)} programs, {len(out)} builtin cases")


if __name__ == "__main__":
    main()
