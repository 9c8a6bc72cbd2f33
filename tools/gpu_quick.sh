#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "== finite 4096"; PROFILE_TRACE=1 timeout 30 stdbuf -oL ./build/probe/profile_worker 10000 4096 2 2>&1 | tail -8
echo "== finite 64"; PROFILE_TRACE=1 timeout 30 stdbuf -oL ./build/probe/profile_worker 10000 64 1 2>&1 | tail -8
echo "== latency"; timeout 60 python tools/latency_probe.py 2>&1 | head -9
echo "== cpp"; timeout 120 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp.log 2>&1; grep -B3 -A3 "FAIL" gpurun_out/cpp.log | head -30; tail -1 gpurun_out/cpp.log
echo "== pytest"; timeout 150 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
echo "== bench"; timeout 300 python bench.py --no-cpu-baseline 2>&1 | tail -1
