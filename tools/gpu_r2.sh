#!/bin/bash
# Round-2 GPU pass: parity suites, gates, device capacity, config-1 bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=gpurun_out/r2.log; : > $L
echo "== pytest -m gpu" >> $L
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3 >> $L
echo "== cpp runtime suite" >> $L
timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "rc $?" >> $L; grep -E "FAIL|cases" gpurun_out/cpp_runtime.log | tail -3 >> $L
echo "== gates ${GATES:---c10 --attention --c6}" >> $L
timeout 600 stdbuf -oL ./build/cpp/gates ${GATES:---c10 --attention --c6} > gpurun_out/gates.log 2> gpurun_out/gates.err; echo "rc $?" >> $L; cat gpurun_out/gates.log >> $L
echo "== finite generation (device capacity)" >> $L
PROFILE_TRACE=1 timeout 60 stdbuf -oL ./build/probe/profile_worker 10000 4096 2 >> $L 2>&1
PROFILE_TRACE=1 timeout 60 stdbuf -oL ./build/probe/profile_worker 10000 64 1 >> $L 2>&1
echo "== untraced capacity: 4096 x2, 64, 65536" >> $L
for e in 4096 4096 64 65536; do timeout 60 ./build/probe/profile_worker 10000 $e 1 2>&1 | head -1 >> $L; done
echo "== config-2 device capacity (finite)" >> $L
GB_C2_FINITE=1 TAG="mixed (all)" timeout 120 python tools/probe/c2.py >> $L 2>&1
echo "== bench config 1" >> $L
timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/qb.json 2> gpurun_out/qb.err; echo "rc $?" >> $L
python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('value',d['value'],'ms',d['ms_per_step'],'submit_ns',d['host_submit_ns_per_task'],'p50',d['p50_submit_to_complete_us'],'p99',d['p99_submit_to_complete_us'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'],'parity',d['parity']['mismatches'])" >> $L 2>&1
cat $L
