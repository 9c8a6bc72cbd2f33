#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for b in 1; do echo "== LP_BCAST=$b"; LP_BCAST=$b timeout 60 python tools/latency_probe.py 2>&1 | sed -n 2,8p; done
BURST_KIND=0 timeout 60 ./build/probe/burst_probe 4 1000 | tail -2
timeout 600 ./build/cpp/gates --c10 | cut -c1-300
export GB_C2_FINITE=1
TAG="mixed" timeout 120 python tools/probe/c2.py
for spec in "0 2 1 0" "0 1 0 0" "2 2 1 2"; do set -- $spec
  TAG="op$1 lay$2 sub$3 dt$4" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=$4 timeout 60 python tools/probe/c2.py; done
python - <<'PY'
import ctypes as C
lib = C.CDLL("paper_2604_17861_b200/lib/libgpuos_bench.so")
lib.gb_set_oracle(b"oracle/liboracle.so")
out = (C.c_double * 32)()
f = lib.gb_config3; f.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for dt in (0, 4):
    f(0, dt, 20, out)
    print("config3", dt, "step_us %.1f phases %s parity mism %d" % (out[0], [round(x, 1) for x in out[5:9]], out[9]))
PY
