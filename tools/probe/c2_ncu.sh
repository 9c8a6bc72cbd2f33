#!/bin/bash
# ncu source-level capture of a finite generation of config-2 row-broadcast adds
# (application replay: the ring lives in host memory, which kernel replay does not restore)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export GB_C2_FINITE=1
for spec in "0 0 0 0" "0 0 0 2"; do set -- $spec
  TAG="op$1 lay$2 sub$3 dt$4" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=$4 timeout 60 python tools/probe/c2.py; done
export C2_TASKS=3000 GB_FORCE_OP=0 GB_FORCE_LAYOUT=2 GB_FORCE_SUB=0 GB_FORCE_DT=0
timeout 900 ncu --set full --import-source on --clock-control none --replay-mode application -k regex:gpuos_worker -c 1 -o gpurun_out/c2_rowbcast -f python tools/probe/c2.py > gpurun_out/c2_ncu.log 2>&1; echo "ncu rc $?"; tail -2 gpurun_out/c2_ncu.log
