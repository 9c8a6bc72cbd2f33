#!/bin/bash
# sdpa task alone: ring + per-op timings at T=128/2048, then one ncu --set full capture of the per-op kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for T in 128 2048; do SDPA_T=$T timeout 60 python tools/probe/sdpa_probe.py; done
SDPA_T=2048 SDPA_INLINE_ONLY=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gpuos_task_kernel -c 1 -o gpurun_out/sdpa_inline python tools/probe/sdpa_probe.py > gpurun_out/sdpa_ncu.log 2>&1; echo ncu rc $?; tail -3 gpurun_out/sdpa_ncu.log
