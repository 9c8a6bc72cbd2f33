#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 60 ./build/probe/body_bench 2>&1 | grep -E "op_add|ew_dense"
PROFILE_TRACE=1 timeout 60 ./build/probe/profile_worker 10000 4096 2 2>&1 | tail -7
PROFILE_TRACE=1 timeout 60 ./build/probe/profile_worker 10000 64 1 2>&1 | tail -7
timeout 60 python tools/latency_probe.py 2>&1 | head -9
timeout 200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
