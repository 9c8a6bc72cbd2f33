"""Pin the oracle (oracle/gpuos_oracle.c) before trusting it (CPU only).

1. Known-answer tests the reference's own suites hold.
2. Bit-exact agreement with the reference kernels themselves
   (oracle/_ref/libref.so, compiled from /root/reference) on every seeded
   F32/F64/I32 case of tests/cases.py, including error codes.
3. The F16/BF16 narrowing restatement against independent converters.
"""
import math

import numpy as np
import pytest

import oracle_lib as ol
from cases import ALL_DTYPES, BF16, F16, F32, F64, I32, Case, Operand, elementwise_cases, linalg_cases, row_cases
from parity import compare, oracle_run, reference_run

REF_DTYPES = (F32, F64, I32)


def T(vals, dtype, shape, strides=None, offset=0):
    return ol.HostTensor(ol.encode(np.asarray(vals, dtype=np.float64), dtype), dtype, shape, strides, offset)


def out(dtype, shape, n=None):
    size = n if n is not None else max(1, int(np.prod(shape)) if len(shape) else 1)
    return ol.HostTensor(ol.encode(np.zeros(size), dtype), dtype, shape)


def read(t):
    return list(ol.decode(t.buf, t.dtype))


# ---------------------------------------------------------------- known answers

@pytest.mark.parametrize("dt", [F32, F64, I32])
def test_relu_pinned(dt):  # test_ops.cpp:106-111
    o = out(dt, [2])
    assert ol.run_oracle("relu", o, [T([-1.0, 2.0], dt, [2])]) == 0
    assert read(o) == [0.0, 2.0]


def test_gelu_zero_and_int_rejected():  # test_ops.cpp:128-141
    o = out(F64, [2])
    assert ol.run_oracle("gelu", o, [T([0.0, 1.0], F64, [2])]) == 0
    assert read(o)[0] == 0.0
    assert abs(read(o)[1] - 0.8411919906082768) < 1e-12
    assert ol.run_oracle("gelu", out(I32, [4]), [T([1, 2, 3, 4], I32, [4])]) == 16


def test_add_broadcast_ones():  # test_ops.cpp:155-162
    o = out(F32, [3, 4])
    assert ol.run_oracle("add", o, [T([1, 1, 1], F32, [3, 1]), T([1, 1, 1, 1], F32, [1, 4])]) == 0
    assert read(o) == [2.0] * 12


def test_add_errors():  # test_ops.cpp:164-179
    a, b64 = T([0] * 4, F32, [4]), T([0] * 4, F64, [4])
    assert ol.run_oracle("add", out(F32, [4]), [a, b64]) == 16
    assert ol.run_oracle("mul", out(F32, [3, 4]), [T([0] * 6, F32, [3, 2]), T([0] * 4, F32, [1, 4])]) == 1
    assert ol.run_oracle("add", out(F32, [4]), [a]) == 13


def test_i32_add():  # test_ops.cpp:204-208
    o = out(I32, [3])
    assert ol.run_oracle("add", o, [T([1, -2, 7], I32, [3]), T([10, 3, -4], I32, [3])]) == 0
    assert read(o) == [11.0, 1.0, 3.0]


def test_softmax_pinned():  # test_ops.cpp:213-220
    for vals in ([0.0, 0.0], [1000.0, 1000.0]):
        o = out(F64, [2])
        assert ol.run_oracle("softmax", o, [T(vals, F64, [2])]) == 0
        assert read(o) == [0.5, 0.5]
    assert ol.run_oracle("softmax", out(F64, [2, 0], 1), [T([0.0], F64, [2, 0], [0, 1])]) == 15


def test_layernorm_pinned():  # test_ops.cpp:255-287
    o = out(F64, [1, 4])
    rc = ol.run_oracle("layernorm", o, [T([2.5] * 4, F64, [1, 4]), T([1.0] * 4, F64, [4]), T([0.0] * 4, F64, [4])])
    assert rc == 0 and read(o) == [0.0] * 4
    o = out(F64, [2, 3])
    rc = ol.run_oracle("layernorm", o, [T([1, 2, 3, -1, 0, 4], F64, [2, 3]), T([0.0] * 3, F64, [3]),
                                        T([1.5, -2.0, 0.25], F64, [3])])
    assert rc == 0 and read(o) == [1.5, -2.0, 0.25, 1.5, -2.0, 0.25]


def test_reduce_pinned():  # test_ops.cpp:331-349
    o = out(F64, [])
    assert ol.run_oracle("reduce_sum", o, [T([1.0, 2.0, 3.0], F64, [3])]) == 0 and read(o) == [6.0]
    o = out(F64, [1])
    assert ol.run_oracle("reduce_max", o, [T([42.5], F64, [1, 1])]) == 0 and read(o) == [42.5]
    z = out(F32, [4])
    empty = T([0.0], F32, [4, 0], [0, 1])
    assert ol.run_oracle("reduce_sum", z, [empty]) == 0 and read(z) == [0.0] * 4
    assert ol.run_oracle("reduce_max", z, [empty]) == 15
    assert ol.run_oracle("reduce_min", z, [empty]) == 15


def test_matmul_pinned():  # test_ops.cpp:389-419
    ident = T([1, 0, 0, 1], F64, [2, 2])
    b = T([1.5, -2.0, 3.0, -7.5], F64, [2, 2])
    o = out(F64, [2, 2])
    assert ol.run_oracle("matmul_small", o, [ident, b]) == 0
    assert read(o) == [1.5, -2.0, 3.0, -7.5]
    big = T(np.zeros(257), F64, [1, 257])
    assert ol.run_oracle("matmul_small", out(F64, [1, 1]), [big, T(np.zeros(257), F64, [257, 1])]) == 18
    assert ol.run_oracle("matmul_small", out(F64, [1, 1]), [big, T(np.zeros(257), F64, [257, 1])],
                         uncapped=True) == 0


def test_sdpa_single_row_copies_v():  # test_ops.cpp:471-479
    q = T([0.3, -0.7], F64, [1, 2])
    k = T([1.0, 2.0], F64, [1, 1, 2])
    v = T([5.0, -6.0], F64, [1, 1, 2])
    o = out(F64, [1, 2])
    assert ol.run_oracle("sdpa", o, [q, k, v]) == 0 and read(o) == [5.0, -6.0]


def test_rope_quarter_turn():  # test_ops.cpp:569-576
    x = T([1.0, 0.0], F64, [1, 2])
    pos = T([math.pi / 4], F64, [1])
    o = out(F64, [1, 2])
    assert ol.run_oracle("rope", o, [x, pos]) == 0
    got = read(o)
    assert abs(got[0] - math.cos(math.pi / 4)) < 1e-14 and abs(got[1] - math.sin(math.pi / 4)) < 1e-14
    assert ol.run_oracle("rope", out(F64, [1, 3]), [T([0, 0, 0], F64, [1, 3]), T([0], F64, [1])]) == 19


def test_kv_append_cursor_and_full():  # test_ops.cpp:638-657
    h, cap, d = 2, 3, 4
    kc, vc = out(F32, [h, cap, d]), out(F32, [h, cap, d])
    nk, nv = T(np.arange(8.0), F32, [h, d]), T(-np.arange(8.0), F32, [h, d])
    assert ol.run_oracle("kv_append", kc, [nk, nv, vc], [1.0]) == 0
    got = np.array(read(kc)).reshape(h, cap, d)
    assert (got[:, 1, :] == np.arange(8.0).reshape(h, d)).all() and (got[:, 0, :] == 0).all()
    assert ol.run_oracle("kv_append", kc, [nk, nv, vc], [3.0]) == 20


def test_program_scale_add():  # test_opcompiler.cpp:226-236, test_runtime.cpp:616-619
    code = [(0, 0, 0.0)]  # placeholder replaced below
    # in0 * 2 + 3 at 4 -> 11; scale_add(2,-1)(1.5) -> 2
    for (p0, p1, x, want) in ((2.0, 3.0, 4.0, 11.0), (2.0, -1.0, 1.5, 2.0)):
        code = [(1, 0, 0.0), (0, 0, p0), (4, 0, 0.0), (0, 0, p1), (2, 0, 0.0), (14, 0, 0.0)]
        o = out(F64, [1])
        assert ol.run_program(code, 1, F64, o, [T([x], F64, [1])]) == 0
        assert read(o) == [want]


def test_broadcast_shapes():  # test_tensor.cpp:76-83
    lib = ol.oracle()
    import ctypes as C
    a = (C.c_int64 * 2)(3, 1)
    b = (C.c_int64 * 2)(1, 4)
    o = (C.c_int64 * 8)()
    r = C.c_int()
    assert lib.orc_broadcast_shapes(a, 2, b, 2, o, C.byref(r)) == 0 and list(o)[:2] == [3, 4]
    a = (C.c_int64 * 2)(2, 3)
    b = (C.c_int64 * 2)(4, 3)
    assert lib.orc_broadcast_shapes(a, 2, b, 2, o, C.byref(r)) == 1


# ---------------------------------------------------------------- oracle == reference

def _ref_cases():
    cs = [c for c in elementwise_cases(dtypes=REF_DTYPES) + row_cases(dtypes=REF_DTYPES) +
          linalg_cases(dtypes=REF_DTYPES) if c.dtype in REF_DTYPES and
          all(o.dtype in REF_DTYPES for o in c.inputs)]
    return cs


@pytest.mark.skipif(ol.reference() is None, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("case", _ref_cases(), ids=lambda c: c.name)
def test_oracle_equals_reference(case: Case):
    rc_o, bufs_o = oracle_run(case)
    rc_r, bufs_r = reference_run(case)
    assert rc_o == rc_r, f"error code oracle {rc_o} vs reference {rc_r}"
    if rc_o != 0:
        return
    for bo, br in zip(bufs_o, bufs_r):
        same = (bo.view(np.uint8) == br.view(np.uint8)).all() or \
            np.array_equal(ol.decode(bo, case.out.dtype), ol.decode(br, case.out.dtype), equal_nan=True)
        assert same, f"oracle and reference differ for {case.name}"


# ---------------------------------------------------------------- F16 / BF16 restatement

def test_f16_narrowing_matches_numpy():
    rng = np.random.default_rng(3)
    vals = np.concatenate([rng.uniform(-70000, 70000, 2000), rng.uniform(-1e-4, 1e-4, 2000),
                           rng.standard_normal(2000) * 1e-6, [65504.0, 65519.99, 65520.0, -65520.0, 6e-8, 5.96e-8,
                                                              2.98e-8, 2.9802322387695312e-08, 0.0, -0.0, np.inf,
                                                              -np.inf]])
    lib = ol.oracle()
    got = np.array([lib.orc_f16_bits(float(v)) for v in vals], dtype=np.uint16)
    want = vals.astype(np.float16).view(np.uint16)
    assert (got == want).all()
    back = np.array([lib.orc_f16_value(int(b)) for b in want])
    assert np.array_equal(back, want.view(np.float16).astype(np.float64))


def test_bf16_narrowing_matches_torch_on_float_exact_values():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(4)
    vals32 = np.concatenate([rng.standard_normal(4000).astype(np.float32) * 1e3,
                             rng.standard_normal(1000).astype(np.float32) * 1e-39,
                             np.array([3.3895314e38, 3.4028235e38, -0.0, 0.0], dtype=np.float32)])
    lib = ol.oracle()
    got = np.array([lib.orc_bf16_bits(float(v)) for v in vals32], dtype=np.uint16)
    want = torch.from_numpy(vals32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert (got == want).all()


def test_bf16_single_rounding_from_double():
    # 1 + 2^-8 + 2^-30 is above the bf16 midpoint 1 + 2^-8: RNE from the exact
    # double rounds up; a detour through float32 would land on the midpoint and
    # round to even (down).  The restatement rounds once.
    lib = ol.oracle()
    x = 1.0 + 2.0 ** -8 + 2.0 ** -30
    assert lib.orc_bf16_bits(x) == 0x3F81
    assert lib.orc_bf16_bits(1.0 + 2.0 ** -8) == 0x3F80  # exact tie -> even
    assert lib.orc_narrow_i32(3e9) == -(2 ** 31) and lib.orc_narrow_i32(-7.9) == -7
