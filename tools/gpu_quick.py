"""First on-GPU check of the ring + persistent worker through the C-ABI."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17861_b200 import abi  # noqa: E402

rng = np.random.default_rng(0)
t0 = time.time()
with abi.Device(0) as d:
    print("open ok", time.time() - t0, "s; alive", d.alive(), "version", d.version())
    n = 4096
    a, b, c = d.alloc(abi.F32, n), d.alloc(abi.F32, n), d.alloc(abi.F32, n)
    x = rng.uniform(-1, 1, n).astype(np.float32)
    y = rng.uniform(-1, 1, n).astype(np.float32)
    a.write(x)
    b.write(y)
    va, vb, vc = (d.view(buf.id, abi.F32, [n]) for buf in (a, b, c))
    t1 = time.time()
    rc = d.run(abi.OP["add"], vc, [va, vb])
    print("ring add rc", rc, "latency(py)", (time.time() - t1) * 1e6, "us")
    got = c.read(np.float32)
    print("add exact:", np.array_equal(got, x + y))
    rc = d.run(abi.OP["mul"], vc, [va, vb])
    print("mul exact:", rc, np.array_equal(c.read(np.float32), x * y))
    rc = d.run(abi.OP["relu"], vc, [va])
    print("relu exact:", rc, np.array_equal(c.read(np.float32), np.where(x < 0, np.float32(0), x)))
    # strided + broadcast
    m = d.alloc(abi.F32, 64 * 64)
    mv = rng.uniform(-1, 1, 64 * 64).astype(np.float32)
    m.write(mv)
    row = d.alloc(abi.F32, 64)
    rv = rng.uniform(-1, 1, 64).astype(np.float32)
    row.write(rv)
    o = d.alloc(abi.F32, 64 * 64)
    rc = d.run(abi.OP["add"], d.view(o.id, abi.F32, [64, 64]),
               [d.view(m.id, abi.F32, [64, 64], [1, 64]), d.view(row.id, abi.F32, [1, 64])])
    want = mv.reshape(64, 64).T + rv[None, :]
    print("transposed+broadcast add:", rc, np.array_equal(o.read(np.float32).reshape(64, 64), want))
    # reduce sum over rows
    r = d.alloc(abi.F32, 64)
    rc = d.run(abi.OP["reduce_sum"], d.view(r.id, abi.F32, [64]), [d.view(m.id, abi.F32, [64, 64])])
    want = np.array([np.float32(sum(float(v) for v in mv[i * 64:(i + 1) * 64])) for i in range(64)])
    print("reduce_sum:", rc, np.array_equal(r.read(np.float32), want))
    # softmax
    rc = d.run(abi.OP["softmax"], d.view(o.id, abi.F32, [64, 64]), [d.view(m.id, abi.F32, [64, 64])])
    xm = mv.reshape(64, 64).astype(np.float64)
    e = np.exp(xm - xm.max(1, keepdims=True))
    want = (e / e.sum(1, keepdims=True)).astype(np.float32)
    print("softmax:", rc, np.max(np.abs(o.read(np.float32).reshape(64, 64) - want)))
    # matmul via ring and via launch
    mm = d.alloc(abi.F32, 64 * 64)
    rc = d.run(abi.OP["matmul_small"], d.view(mm.id, abi.F32, [64, 64]),
               [d.view(m.id, abi.F32, [64, 64]), d.view(m.id, abi.F32, [64, 64], [1, 64])])
    A = mv.reshape(64, 64).astype(np.float64)
    print("matmul:", rc, np.max(np.abs(mm.read(np.float32).reshape(64, 64) - (A @ A.T).astype(np.float32))))
    rc = d.run_inline(abi.OP["add"], vc, [va, vb])
    print("inline add:", rc, np.array_equal(c.read(np.float32), x + y))
    # error paths
    print("arity error:", abi.ERRORS[d.run(abi.OP["add"], vc, [va])])
    print("not installed:", abi.ERRORS[d.run(40, vc, [va])])
    print("out of range:", abi.ERRORS[d.run(5000, vc, [va])])
    # throughput via python producer (upper bound is python)
    N = 20000
    ts = [d.make_task(abi.OP["add"], vc, [va, vb], cell=False) for _ in range(N)]
    s0 = d.peek().processed
    t1 = time.time()
    for t in ts:
        d.submit(t)
    d.wait_processed(s0 + N)
    dt = time.time() - t1
    print(f"python-producer throughput: {N / dt:.0f} tasks/s")
    st = d.stats()
    print("stats processed", st.processed, "failed", st.failed, "canary", st.canary_hits, "torn", st.torn_reads)
    tr = d.trace(100)
    print("trace records", len(tr), tr[-1].exec_ns if tr else None)
    print("peek", d.peek().head, d.peek().tail, d.peek().processed)
print("closed ok")
