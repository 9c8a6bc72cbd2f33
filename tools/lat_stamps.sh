#!/bin/bash
# Depth-1 latency phases with the product library, then the clock64 bisection
# of the GPUOS_LAT_STAMPS build (make lat-debug) on one worker.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 60 python tools/latency_probe.py 2>&1 | sed -n 2,8p
cp build/dbg/libgpuos_cuda.so paper_2604_17861_b200/lib/libgpuos_cuda.so
LP_WORKERS=1 timeout 60 python tools/latency_probe.py 2>&1 | grep "^LAT" | sed -n 4,8p
