#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
echo "== finite 4096"; PROFILE_TRACE=1 timeout 30 stdbuf -oL ./build/probe/profile_worker 10000 4096 2 2>&1 | tail -8
echo "== finite 65536"; timeout 30 stdbuf -oL ./build/probe/profile_worker 1000 65536 2 2>&1 | tail -3
echo "== latency"; timeout 60 python tools/latency_probe.py 2>&1 | head -9
echo "== pytest"; timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
echo "== c2 contiguous add"; TAG=add-contig GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py
echo "== bench"; timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); c=d['configs']
print(d['value'], d['p50_submit_to_complete_us'], d['roofline']['frac'], d['e2e']['value'])
for k,v in c.items(): print(k, {kk: vv for kk, vv in v.items() if kk != 'workload'})"
