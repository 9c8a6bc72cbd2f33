#!/bin/bash
# A/B: completer release fence at gpu scope (product) vs sys scope (build/fsys)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
cp paper_2604_17861_b200/lib/libgpuos_cuda.so /tmp/lib_gpu.so
for v in gpu sys gpu sys; do
  if [ $v = gpu ]; then cp /tmp/lib_gpu.so paper_2604_17861_b200/lib/libgpuos_cuda.so; else cp build/fsys/libgpuos_cuda.so paper_2604_17861_b200/lib/libgpuos_cuda.so; fi
  echo "== fence.release.$v"
  for e in 4096 64; do timeout 60 ./build/probe/profile_worker 10000 $e 1 2>&1 | head -1; done
  timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline | python -c "import json,sys;d=json.load(sys.stdin);print('value',d['value'],'p50',d['p50_submit_to_complete_us'],'p99',d['p99_submit_to_complete_us'])"
done
cp /tmp/lib_gpu.so paper_2604_17861_b200/lib/libgpuos_cuda.so
