#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 120 ./build/probe/burst_probe 6 1000
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 400 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?"; grep -E "cases|FAIL" gpurun_out/cpp_runtime.log
for e in 4096 64; do timeout 60 ./build/probe/profile_worker 10000 $e 1 2>&1 | head -1; done
python - <<'PY'
import ctypes as C
lib = C.CDLL("paper_2604_17861_b200/lib/libgpuos_bench.so")
lib.gb_set_oracle(b"oracle/liboracle.so")
out = (C.c_double * 32)()
for fn in ("gb_config3", "gb_config3_fenced"):
    f = getattr(lib, fn); f.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for dt in (0, 4):
        f(0, dt, 20, out)
        print(fn, dt, "step_us %.1f phases %s parity mism %d" % (out[0], [round(x, 1) for x in out[5:9]], out[9]))
PY
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-configs --no-cpu-baseline | python -c "import json,sys;d=json.load(sys.stdin);print(d['value'],d['host_submit_ns_per_task'],d['p50_submit_to_complete_us'],d['p99_submit_to_complete_us'],d['e2e']['value'])"; done
