# Config-2 device cost per (op, layout, sub-layout, dtype): finite generations
# over a prepublished ring (GB_C2_FINITE), so the host producer is out of the
# loop and tasks/s + algorithmic GB/s are the worker kernel's own.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export GB_C2_FINITE=1
TAG="mixed (all)" timeout 120 python tools/probe/c2.py
for op in 0 1 2 3; do for lay in 0 1 2; do for sub in 0 1; do
  TAG="op$op lay$lay sub$sub dt0" GB_FORCE_OP=$op GB_FORCE_LAYOUT=$lay GB_FORCE_SUB=$sub GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py
done; done; done
for dt in 1 2 3; do for op in 0 3; do TAG="op$op lay0 dt$dt" GB_FORCE_OP=$op GB_FORCE_LAYOUT=0 GB_FORCE_DT=$dt timeout 60 python tools/probe/c2.py; done; done
