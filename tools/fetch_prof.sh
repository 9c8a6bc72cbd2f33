#!/bin/bash
# Fetcher hand-off cycle profile: the GPUOS_FETCH_PROF build drains a
# prepublished ring (finite generation) and CTAs 0..3 print per-segment cycles.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_2604_17861_b200/lib/libgpuos_cuda.so /tmp/lib_prod.so
cp build/fprof/libgpuos_cuda.so paper_2604_17861_b200/lib/libgpuos_cuda.so
for e in 4096 64; do echo "== $e"; timeout 60 ./build/probe/profile_worker 10000 $e 1 2>&1 | grep -E "FPROF|tasks_per_s"; done
cp /tmp/lib_prod.so paper_2604_17861_b200/lib/libgpuos_cuda.so
