#!/bin/bash
# Quick GPU-box pass for producer/step work: submit-cost breakdown, the C++
# runtime suite, then config 1 only (no configs 2-5, no CPU baseline).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
echo "== submit cost"; timeout 120 ./build/probe/submit_cost 2>&1 | tail -7
echo "== cpp"; timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp.log 2>&1; echo rc $?; tail -1 gpurun_out/cpp.log
echo "== bench config 1"
for i in 1 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/qb.json 2> gpurun_out/qb.err; echo "rc $?"
python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('value',d['value'],'ms',d['ms_per_step'],'submit_ns',d['host_submit_ns_per_task'],'p50',d['p50_submit_to_complete_us'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],'parity',d['parity']['mismatches'])"
done
