#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=gpurun_out/probe.log; : > $L
echo "== profile_worker" >> $L
for cfg in "10000 64" "10000 4096" "2500 16384"; do
  timeout 60 stdbuf -oL ./build/probe/profile_worker $cfg 3 >> $L 2>&1 || echo "rc $? ($cfg)" >> $L
done
echo "== submit_cost" >> $L
timeout 60 stdbuf -oL ./build/probe/submit_cost 2>&1 | tail -6 >> $L
echo "== cpp" >> $L
timeout 120 stdbuf -oL ./build/cpp/test_runtime 2>&1 | tail -4 >> $L
echo "== pytest" >> $L
timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> $L
echo "== bench" >> $L
timeout 300 python bench.py --no-cpu-baseline >> $L 2>&1
cat $L
