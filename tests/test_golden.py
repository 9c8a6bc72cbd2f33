"""The oracle against fixtures produced by the reference itself
(tests/golden/make_golden.py): runs anywhere, including boxes without
/root/reference, so the checker stays pinned on the GPU box too."""
import json
import os

import numpy as np
import pytest

import oracle_lib as ol
from cases import Case, Operand

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "builtins.json")) as f:
    BUILTINS = json.load(f)
with open(os.path.join(HERE, "golden", "programs.json")) as f:
    PROGRAMS = json.load(f)


def _tensor(spec):
    buf = np.frombuffer(bytes.fromhex(spec["data"]), dtype=ol.NP[spec["dtype"]]).copy()
    return ol.HostTensor(buf, spec["dtype"], spec["shape"], spec["strides"], spec["offset"])


@pytest.mark.parametrize("fx", BUILTINS, ids=lambda f: f["name"])
def test_oracle_matches_reference_fixture(fx):
    ins = [_tensor(s) for s in fx["inputs"]]
    o = fx["out"]
    out = ol.HostTensor(np.zeros(o["size"], dtype=ol.NP[o["dtype"]]), o["dtype"], o["shape"], o["strides"],
                        o["offset"])
    rc = ol.run_oracle(fx["op"], out, ins, fx["scalars"])
    assert rc == fx["code"]
    if rc:
        return
    got = [out.buf] + ([ins[2].buf] if fx["op"] == "kv_append" else [])
    for g, hexs in zip(got, fx["results"]):
        assert g.tobytes() == bytes.fromhex(hexs), fx["name"]


def test_fixture_coverage():
    ops = {f["op"] for f in BUILTINS}
    assert {"add", "mul", "relu", "gelu", "softmax", "layernorm", "reduce_sum", "reduce_max", "reduce_min",
            "matmul_small", "vecmat", "sdpa", "rope", "kv_append"} <= ops
    assert len(PROGRAMS) == 9
