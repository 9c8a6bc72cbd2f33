#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?"; grep -B1 -A3 "fused chains equal the oracle" gpurun_out/cpp_runtime.log | head; grep cases gpurun_out/cpp_runtime.log
export GB_C2_FINITE=1
for dt in 0 1 2 3; do TAG="mixed dt$dt" GB_FORCE_DT=$dt timeout 120 python tools/probe/c2.py; done
for op in 0 1 2 3; do TAG="mixed op$op" GB_FORCE_OP=$op timeout 120 python tools/probe/c2.py; done
