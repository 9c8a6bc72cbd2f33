#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for T in 128 2048; do SDPA_T=$T timeout 60 python tools/probe/sdpa_probe.py; done
timeout 300 ./build/cpp/gates --attention
python - <<'PY'
import ctypes as C
lib = C.CDLL("paper_2604_17861_b200/lib/libgpuos_bench.so")
out = (C.c_double * 32)()
lib.gb_swap_latency.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
lib.gb_swap_latency(0, 200000, 16, out)
print("swap latency: entry->first new p50 %.1f us max %.1f | return->first new p50 %.1f | call %.1f us | swaps %d | late old %d | %.0f tasks/s" % tuple(out[i] for i in range(7)))
PY
