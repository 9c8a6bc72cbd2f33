#!/bin/bash
# Device capacity vs task size (dense f32 add, aligned) and the effect of
# 16-byte alignment on the config-2 stream (GB_FORCE_ALIGN).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for e in 1024 4096 16384 65536; do timeout 90 ./build/probe/profile_worker 10000 $e 1 2>&1 | head -1; done
export GB_C2_FINITE=1
for a in 0 1; do
  if [ $a = 1 ]; then export GB_FORCE_ALIGN=1; fi
  TAG="align=$a add contiguous f32" GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 timeout 120 python tools/probe/c2.py
  TAG="align=$a add contiguous bf16" GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=2 timeout 120 python tools/probe/c2.py
  TAG="align=$a reduce contiguous f32" GB_FORCE_OP=3 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 timeout 120 python tools/probe/c2.py
  TAG="align=$a mixed" timeout 120 python tools/probe/c2.py
done
