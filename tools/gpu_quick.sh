#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "== pytest all"; timeout 200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
echo "== cpp"; timeout 120 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp.log 2>&1; grep -B3 -A3 "FAIL" gpurun_out/cpp.log | head -30; tail -1 gpurun_out/cpp.log
echo "== bench configs"; timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); c=d['configs']
print(d['value'], d['p50_submit_to_complete_us'])
for k,v in c.items(): print(k, {kk: vv for kk, vv in v.items() if kk != 'workload'})"
