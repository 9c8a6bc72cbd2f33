#!/bin/bash
# L1 vs shared-memory carveout: the executors' spilled stack frames live in L1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cv in 100 72 100 72; do
  echo "== carveout $cv"
  export GPUOS_CARVEOUT=$cv
  timeout 120 ./build/probe/burst_probe 4 1000 | tail -2
  timeout 60 ./build/probe/profile_worker 10000 4096 1 2>&1 | head -1
  GB_C2_FINITE=1 TAG="c2 mixed" timeout 120 python tools/probe/c2.py
done
