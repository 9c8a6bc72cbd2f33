#!/bin/bash
# A/B of device capacity: product library vs build/nobulk (register-path elementwise).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_2604_17861_b200/lib/libgpuos_cuda.so /tmp/lib_a.so
for v in A B A B; do
  if [ $v = A ]; then cp /tmp/lib_a.so paper_2604_17861_b200/lib/libgpuos_cuda.so; else cp build/nobulk/libgpuos_cuda.so paper_2604_17861_b200/lib/libgpuos_cuda.so; fi
  echo "== $v"
  timeout 60 ./build/probe/profile_worker 10000 4096 1 2>&1 | head -1
  timeout 60 ./build/probe/profile_worker 10000 65536 1 2>&1 | head -1
  timeout 60 ./build/probe/profile_worker 10000 64 1 2>&1 | head -1
  GB_C2_FINITE=1 GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 TAG="c2 add contiguous f32" timeout 120 python tools/probe/c2.py 2>&1
  GB_C2_FINITE=1 TAG="c2 mixed" timeout 120 python tools/probe/c2.py 2>&1
done
cp /tmp/lib_a.so paper_2604_17861_b200/lib/libgpuos_cuda.so
