#!/bin/bash
# One GPU-box pass: parity suites, smoke, latency phases, bench.  Logs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
L=gpurun_out/check.log; : > $L
echo "== pytest -m gpu" >> $L
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3 >> $L
echo "== cpp runtime suite" >> $L
timeout 200 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "rc $?" >> $L; tail -2 gpurun_out/cpp_runtime.log >> $L
echo "== smoke" >> $L
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "== finite generation (device capacity)" >> $L
PROFILE_TRACE=1 timeout 60 stdbuf -oL ./build/probe/profile_worker 10000 4096 2 >> $L 2>&1
PROFILE_TRACE=1 timeout 60 stdbuf -oL ./build/probe/profile_worker 10000 64 1 >> $L 2>&1
echo "== latency phases" >> $L
timeout 120 python tools/latency_probe.py >> $L 2>&1
echo "== bench" >> $L
timeout 400 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> $L
cat gpurun_out/bench.json >> $L
cat $L
