#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
LP_BCAST=1 timeout 60 python tools/latency_probe.py 2>&1 | sed -n 5,5p
timeout 60 python tools/latency_probe.py 2>&1 | sed -n 5,5p
export GB_C2_FINITE=1
TAG="mixed" timeout 120 python tools/probe/c2.py
TAG="mixed" timeout 120 python tools/probe/c2.py
for spec in "0 2 1 0" "0 1 1 0" "0 2 0 0"; do set -- $spec
  TAG="op$1 lay$2 sub$3 dt$4" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=$4 timeout 60 python tools/probe/c2.py; done
