cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=mixed timeout 60 python tools/probe/c2.py
for spec in "0 1 1" "0 2 0" "2 1 1" "2 2 0" "3 0 0" "3 1 0"; do set -- $spec; TAG="op$1 lay$2 sub$3" GB_FORCE_OP=$1 GB_FORCE_LAYOUT=$2 GB_FORCE_SUB=$3 GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py; done
timeout 300 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
