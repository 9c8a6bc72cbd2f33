#!/bin/bash
# One GPU-box pass: parity suites, smoke, bench.  Logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?" >> gpurun_out/cpp_runtime.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_gpu.log gpurun_out/cpp_runtime.log gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
