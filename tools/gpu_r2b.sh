#!/bin/bash
# fence test + config 3 both variants + sdpa probe
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 400 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp_runtime.log 2>&1; echo "cpp rc $?"; grep -E "FAIL|cases|fence" gpurun_out/cpp_runtime.log | tail -5
python - <<'PY'
import ctypes as C, os, json
lib = C.CDLL("paper_2604_17861_b200/lib/libgpuos_bench.so")
lib.gb_set_oracle(b"oracle/liboracle.so")
out = (C.c_double * 32)()
for fn in ("gb_config3", "gb_config3_fenced"):
    f = getattr(lib, fn); f.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for dt in (0, 4):
        f(0, dt, 20, out)
        print(fn, dt, "step_us %.1f phases %s parity mism %d checked %d" % (out[0], [round(x, 1) for x in out[5:9]], out[9], out[10]))
PY
bash tools/probe/sdpa_ncu.sh
