#!/bin/bash
# Round-end pass: parity suites, C++ suites, every gate, smoke, then the full bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
L=gpurun_out/final.log; : > $L
echo "== pytest -m gpu" >> $L; timeout 500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2 >> $L
echo "== cpp runtime suite" >> $L; timeout 400 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "rc $?" >> $L; grep -E "FAIL|cases|TaskQueue|fused chains|live ring|f32:|f64:" gpurun_out/cpp_runtime.log >> $L
echo "== gates" >> $L; timeout 900 stdbuf -oL ./build/cpp/gates > gpurun_out/gates.log 2> gpurun_out/gates.err; echo "rc $?" >> $L; cat gpurun_out/gates.log >> $L
echo "== smoke" >> $L; timeout 120 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1
echo "== bench" >> $L; timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "rc $?" >> $L
cat $L
