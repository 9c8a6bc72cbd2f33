#!/bin/bash
# ncu --set full of one finite worker generation serving a depth-1 task stream
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 60 python tools/probe/lat_ncu.py; echo "plain rc $?"
timeout 900 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:gpuos_worker -c 1 -o gpurun_out/worker_lat -f python tools/probe/lat_ncu.py > gpurun_out/ncu_lat_run.log 2>&1; echo "ncu rc $?"
tail -5 gpurun_out/ncu_lat_run.log
