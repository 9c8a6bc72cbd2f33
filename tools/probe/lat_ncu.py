"""Depth-1 task stream against ONE finite worker generation, for ncu.

Under ncu the worker launch blocks until the kernel exits, so thread A starts
the generation (GPUOS_DEFER_START=1) while thread B feeds tasks one at a time
through host memory only (ring publish + completion-cell spin, no CUDA calls)
and finally publishes the shutdown sentinel, which ends the generation.
"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["GPUOS_DEFER_START"] = "1"
from paper_2604_17861_b200 import abi  # noqa: E402

n = int(os.environ.get("LP_N", "4096"))
iters = int(os.environ.get("LP_ITERS", "400"))
d = abi.Device(0, telemetry=False, num_workers=int(os.environ.get("LP_WORKERS", "1")))
a, b, c = d.alloc(abi.F32, n), d.alloc(abi.F32, n), d.alloc(abi.F32, n)
a.write(np.ones(n, np.float32))
b.write(np.ones(n, np.float32))
va, vb, vc = (d.view(x.id, abi.F32, [n]) for x in (a, b, c))
tasks = [d.make_task(abi.OP["add"], vc, [va, vb]) for _ in range(iters)]
stop = d.make_task(abi.OP["add"], vc, [va, vb], flags=abi.FLAG_SHUTDOWN, cell=False)
lat = []


def feed():
    time.sleep(0.5)
    for t in tasks:
        t0 = time.perf_counter()
        d.submit(t)
        d.wait_cell(t, timeout=60.0)
        lat.append((time.perf_counter() - t0) * 1e6)
    d.submit(stop)


th = threading.Thread(target=feed)
th.start()
rc = d.start()
th.join()
print("start rc", rc, "p50 us", np.percentile(lat[50:], 50))
d.close()
