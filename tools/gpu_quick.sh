#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "== pytest"; timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== cpp"; timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp.log 2>&1; grep -B3 -A3 "FAIL" gpurun_out/cpp.log | head -20; tail -1 gpurun_out/cpp.log
echo "== latency"; timeout 60 python tools/latency_probe.py 2>&1 | sed -n 2,8p
echo "== body"; timeout 60 ./build/probe/body_bench | grep "idle=    0" | grep "n=  4096\|n=    64"
echo "== finite"; timeout 30 ./build/probe/profile_worker 10000 4096 2 | tail -2 | head -1
echo "== bench"; timeout 200 python bench.py --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['host_submit_ns_per_task'], d['p50_submit_to_complete_us'], d['p99_submit_to_complete_us'], d['parity'])"
