cd "${GRAFT_REPO_ROOT:-/root/repo}"
for op in 0 1 2 3; do for lay in 0 1 2; do for sub in 0 1; do
  TAG="op$op lay$lay sub$sub dt0" GB_FORCE_OP=$op GB_FORCE_LAYOUT=$lay GB_FORCE_SUB=$sub GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py
done; done; done
for dt in 1 2 3; do TAG="op0 lay0 dt$dt" GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=$dt timeout 60 python tools/probe/c2.py; done
