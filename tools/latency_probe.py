"""Phase breakdown of submit->complete on the device path (trace stamps)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_17861_b200 import abi  # noqa: E402


def summarize(name, ph, t_host=None):
    a = np.array([[p.enqueue_ns, p.ticket_ns, p.seen_ns, p.dequeue_ns, p.end_ns, p.done_ns] for p in ph],
                 dtype=np.float64)
    if len(a) == 0:
        print(name, "no records")
        return
    d = {
        "enq->seen": a[:, 2] - a[:, 0],
        "seen->deq": a[:, 3] - a[:, 2],
        "deq->wake": np.array([p.reserved for p in ph], dtype=np.float64),
        "deq->end(exec)": a[:, 4] - a[:, 3],
        "end->done": a[:, 5] - a[:, 4],
        "ticket->seen": a[:, 2] - a[:, 1],
    }
    print(f"== {name}: {len(a)} records")
    for k, v in d.items():
        print(f"  {k:16s} p50 {np.percentile(v, 50) / 1e3:9.2f} us  p90 {np.percentile(v, 90) / 1e3:9.2f} us")
    if t_host is not None:
        print(f"  host submit->wait p50 {np.percentile(t_host, 50):.2f} us p99 {np.percentile(t_host, 99):.2f} us")


n = int(os.environ.get("LP_N", "4096"))
with abi.Device(0, telemetry=True, num_workers=int(os.environ.get("LP_WORKERS", "0"))) as d:
    a, b, c = d.alloc(abi.F32, n), d.alloc(abi.F32, n), d.alloc(abi.F32, n)
    a.write(np.ones(n, np.float32))
    b.write(np.ones(n, np.float32))
    va, vb, vc = (d.view(x.id, abi.F32, [n]) for x in (a, b, c))
    if os.environ.get("LP_BCAST"):  # rank-0 broadcast second input: an extended slot, the general path
        vb = d.view(b.id, abi.F32, [], [])
    lat = []
    for i in range(300):
        t = d.make_task(int(os.environ.get("LP_OP", abi.OP["add"])), vc, [va, vb])
        t0 = time.perf_counter()
        d.submit(t)
        d.wait_cell(t)
        lat.append((time.perf_counter() - t0) * 1e6)
    summarize("queue depth 1", d.phases()[-250:], np.array(lat[50:]))
    N = 20000
    ts = [d.make_task(abi.OP["add"], vc, [va, vb], cell=False) for _ in range(N)]
    s0 = d.peek().processed
    t0 = time.perf_counter()
    for t in ts:
        d.submit(t)
    d.wait_processed(s0 + N)
    dt = time.perf_counter() - t0
    print(f"burst {N}: {N / dt:.0f} tasks/s (python producer)")
    summarize("burst", d.phases()[-N:])
    st = d.stats()
    print("torn", st.torn_reads, "stalls", st.stalls, "canary", st.canary_hits)
