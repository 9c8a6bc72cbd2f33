#!/bin/bash
# smoke (plain and under ncu's launch-list pass), launch list of a finite generation, burst-after-idle timeline
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "smoke-ncu rc $?"; tail -1 gpurun_out/smoke_ncu.log; grep -c gpuos_worker_kernel gpurun_out/smoke_launches.csv
GPUOS_DEFER_START=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv ./build/probe/profile_worker 10000 4096 1 > gpurun_out/ncu_launch_run.log 2>&1; echo "launch list rc $?"; grep -c worker gpurun_out/ncu_launches.csv
timeout 120 ./build/probe/burst_probe 6 1000
timeout 120 python tools/latency_probe.py 2>&1 | head -9
