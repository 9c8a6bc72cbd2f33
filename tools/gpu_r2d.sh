#!/bin/bash
# parity suites + config-2 focus + config-1 bench with the lean per-op baseline
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 400 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?"; grep -E "FAIL|cases|native" gpurun_out/cpp_runtime.log | tail -4
export GB_C2_FINITE=1
TAG="mixed" timeout 120 python tools/probe/c2.py
for spec in "0 0 0 0" "0 0 0 2" "0 1 1 0" "0 2 0 0" "2 2 0 0" "0 1 0 0" "0 2 1 0" "1 1 1 1" "0 2 0 2"; do set -- $spec
  TAG="op$1 lay$2 sub$3 dt$4" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=$4 timeout 60 python tools/probe/c2.py; done
unset GB_C2_FINITE
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/full.json 2> gpurun_out/full.err; echo "bench rc $?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/full.json"))
print("value", d["value"], "p50", d["p50_submit_to_complete_us"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"])
print("per-op", d["baseline_per_op_launch"]["value"], "lean", d["baseline_per_op_launch_lean"]["value"], d["baseline_per_op_launch_lean"]["speedup"])
for k, v in d["configs"].items():
    print(k, json.dumps({kk: vv for kk, vv in v.items() if kk not in ("workload",)})[:420])
PY
