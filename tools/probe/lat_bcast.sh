#!/bin/bash
# depth-1 phases and clock64 bisection for a dense add vs a rank-0-broadcast add (general path)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for b in "" 1; do echo "== LP_BCAST=$b"; LP_BCAST=$b timeout 60 python tools/latency_probe.py 2>&1 | sed -n 2,8p; done
cp paper_2604_17861_b200/lib/libgpuos_cuda.so /tmp/lib_prod.so
cp build/dbg/libgpuos_cuda.so paper_2604_17861_b200/lib/libgpuos_cuda.so
for b in "" 1; do echo "== dbg LP_BCAST=$b"; LP_BCAST=$b LP_WORKERS=1 timeout 60 python tools/latency_probe.py 2>&1 | grep "^LAT" | sed -n 4,8p; done
cp /tmp/lib_prod.so paper_2604_17861_b200/lib/libgpuos_cuda.so
