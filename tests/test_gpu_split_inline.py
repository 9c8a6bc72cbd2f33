"""GPU checks for two worker fast paths, through the task ring.

* Idle split: with nothing else published, a task of >= 2048 elements runs as
  two halves on the CTA's two executor groups and completes once.
* Inline dense f32 add/mul: after the table resolve, a builtin add or mul over
  planned, 16-byte-aligned dense f32 views runs inline in the executor with
  f32-native arithmetic. A misaligned view takes the jump table instead.

Expected values come from numpy's IEEE f32 + and *. They equal the reference's
double evaluation narrowed once (ops.hpp:133-194), because double rounding is
innocuous for + and * from f32 (53 >= 2*24 + 2). So these tests also pin that
claim on special values: signed zeros, denormals, infinities and NaN.
Sizes straddle the split threshold (2048) and the 4-element vector tail.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SIZES = [1, 3, 5, 2047, 2048, 2049, 4096, 4097, 65537]


def _specials(rng, n):
    x = rng.standard_normal(n).astype(np.float32) * np.float32(1e3)
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.17549435e-38, 3.4028235e38, -3.4028235e38],
                  dtype=np.float32)
    k = min(n, sp.size * 4)
    idx = rng.choice(n, size=k, replace=False)
    x[idx] = np.resize(sp, k)
    return x


def _same_bits(got, want):
    both_nan = np.isnan(got) & np.isnan(want)
    return np.all((got.view(np.uint32) == want.view(np.uint32)) | both_nan)


@pytest.mark.parametrize("offset", [0, 1], ids=["aligned", "misaligned"])
@pytest.mark.parametrize("op", ["add", "mul", "relu"])
@pytest.mark.parametrize("n", SIZES)
def test_dense_f32_fast_paths_bit_exact(device, op, n, offset):
    from paper_2604_17861_b200 import abi
    rng = np.random.default_rng(n * 7 + offset * 3 + len(op))
    total = n + offset
    a_np, b_np = _specials(rng, total), _specials(rng, total)
    a, b, c = (device.alloc(abi.F32, total) for _ in range(3))
    a.write(a_np)
    b.write(b_np)
    c.write(np.full(total, np.float32(7.0)))
    va, vb, vc = (device.view(x.id, abi.F32, [n], offset=offset) for x in (a, b, c))
    inputs = [va] if op == "relu" else [va, vb]
    rc = device.run(abi.OP[op], vc, inputs)
    assert abi.ERRORS[rc] == "Ok"
    got = c.read(np.float32)
    x, y = a_np[offset:], b_np[offset:]
    with np.errstate(over="ignore", invalid="ignore"):
        want = x + y if op == "add" else x * y
    if op == "relu":  # v < 0 ? 0 : v keeps -0.0 and NaN (ops.hpp:188)
        want = np.where(x < 0, np.float32(0.0), x)
    assert _same_bits(got[offset:], want.astype(np.float32)), f"{op} n={n} offset={offset}"
    assert np.all(got[:offset] == np.float32(7.0)), "write before the view"
    for buf in (a, b, c):
        device.free(buf)


def test_split_completes_each_task_once(device):
    """Back-to-back idle tasks above the split threshold: each completion cell
    turns terminal exactly once with Ok, and the processed count advances by
    exactly the number of tasks."""
    from paper_2604_17861_b200 import abi
    n = 8192
    a, b, c = (device.alloc(abi.F32, n) for _ in range(3))
    a.write(np.arange(n, dtype=np.float32))
    b.write(np.ones(n, np.float32))
    va, vb, vc = (device.view(x.id, abi.F32, [n]) for x in (a, b, c))
    before = device.peek().processed
    for _ in range(64):
        assert abi.ERRORS[device.run(abi.OP["add"], vc, [va, vb])] == "Ok"
    device.wait_processed(before + 64)
    assert device.peek().processed == before + 64
    assert np.array_equal(c.read(np.float32), np.arange(n, dtype=np.float32) + np.float32(1))
    for buf in (a, b, c):
        device.free(buf)
