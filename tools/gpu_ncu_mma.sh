#!/bin/bash
# Tensor-pipe evidence: finite generation of 2,000 bf16 matmul_small tasks.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GPUOS_DEFER_START=1
PW_OP=matmul_bf16 timeout 120 ./build/probe/profile_worker 2000 4096 2
PW_OP=matmul_bf16 timeout 900 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:gpuos_worker -c 1 -o gpurun_out/worker_mma -f ./build/probe/profile_worker 2000 4096 1 > gpurun_out/ncu_mma_run.log 2>&1; echo "ncu rc $?"
