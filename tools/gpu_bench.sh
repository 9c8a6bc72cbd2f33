#!/bin/bash
# One bench pass on the GPU box: host facts, then bench.py (args in BENCH_ARGS).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
free -g | head -2; nproc; lscpu | grep "Model name"
SECONDS=0; timeout ${BENCH_TIMEOUT:-1200} python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $? in ${SECONDS}s"
tail -5 gpurun_out/bench.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read())
c = d.pop("configs") or {}
print(json.dumps(d)[:1500])
for k, v in c.items():
    print(k, json.dumps(v)[:900])
PY
