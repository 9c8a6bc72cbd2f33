#!/bin/bash
# ncu evidence for the worker kernel: launch list + one --set full capture of a
# finite generation (GPUOS_DEFER_START: no resident generation before it).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
N=${NCU_TASKS:-10000}
export GPUOS_DEFER_START=1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv ./build/probe/profile_worker $N 4096 1 > gpurun_out/ncu_launch_run.log 2>&1; echo "launch list rc $?"
timeout 1200 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:gpuos_worker -c 1 -o gpurun_out/worker_full -f ./build/probe/profile_worker $N 4096 1 > gpurun_out/ncu_full_run.log 2>&1; echo "full rc $?"
tail -3 gpurun_out/ncu_full_run.log
grep -i worker gpurun_out/ncu_launches.csv | head -5
