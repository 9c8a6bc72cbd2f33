#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?"; grep -E "cases|FAIL" gpurun_out/cpp_runtime.log
export GB_C2_FINITE=1
TAG="mixed" timeout 120 python tools/probe/c2.py
for dt in 3 0; do TAG="mixed dt$dt" GB_FORCE_DT=$dt timeout 120 python tools/probe/c2.py; done
for spec in "0 1 1 3" "1 0 0 3" "0 2 0 3"; do set -- $spec
  TAG="op$1 lay$2 sub$3 dt$4" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=$4 timeout 60 python tools/probe/c2.py; done
