"""Decode-attention sdpa task alone (h=4, d=64, context T): ring path and
per-op launch path, device body time from the trace; for ncu run with
SDPA_INLINE_ONLY=1 (no live generation)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2604_17861_b200 import abi  # noqa: E402

T = int(os.environ.get("SDPA_T", "2048"))
h, d = 4, 64
inline_only = bool(os.environ.get("SDPA_INLINE_ONLY"))
with abi.Device(0, telemetry=True, defer_start=inline_only) as dev:
    q, k, v, o = dev.alloc(abi.F32, h * d), dev.alloc(abi.F32, h * T * d), dev.alloc(abi.F32, h * T * d), dev.alloc(abi.F32, h * d)
    rng = np.random.default_rng(1)
    for b, n in ((q, h * d), (k, h * T * d), (v, h * T * d)):
        b.write(rng.uniform(-1, 1, n).astype(np.float32))
    vq, vo = dev.view(q.id, abi.F32, [h, d]), dev.view(o.id, abi.F32, [h, d])
    vk, vv = dev.view(k.id, abi.F32, [h, T, d]), dev.view(v.id, abi.F32, [h, T, d])
    for i in range(5 if inline_only else 20):
        t0 = time.perf_counter()
        rc = dev.run_inline(abi.OP["sdpa"], vo, [vq, vk, vv])
        dt_inline = (time.perf_counter() - t0) * 1e6
    print(f"T={T} inline rc {rc} launch+sync {dt_inline:.1f} us")
    if not inline_only:
        lat = []
        for i in range(20):
            t0 = time.perf_counter()
            rc = dev.run(abi.OP["sdpa"], vo, [vq, vk, vv])
            lat.append((time.perf_counter() - t0) * 1e6)
        ph = dev.phases()[-10:]
        ex = sorted((p.end_ns - p.dequeue_ns) / 1e3 for p in ph)
        print(f"T={T} ring rc {rc} submit->wait p50 {np.median(lat):.1f} us, device exec p50 {ex[len(ex)//2]:.1f} us")
