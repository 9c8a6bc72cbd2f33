#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ./build/cpp/gates --c10 | cut -c1-420
python - <<'PY'
import ctypes as C
lib = C.CDLL("paper_2604_17861_b200/lib/libgpuos_bench.so")
lib.gb_set_oracle(b"oracle/liboracle.so")
out = (C.c_double * 32)()
for fn in ("gb_config3", "gb_config3_fenced"):
    f = getattr(lib, fn); f.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for dt in (0, 4):
        f(0, dt, 20, out)
        print(fn, dt, "step_us %.1f phases %s parity mism %d checked %d bitexact %.6f" % (out[0], [round(x, 1) for x in out[5:9]], out[9], out[10], out[12]))
PY
