cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=batch-mixed timeout 60 python tools/probe/c2.py
TAG=batch-contig GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py
cp paper_2604_17861_b200/lib/libgpuos_cuda_nobatch.so paper_2604_17861_b200/lib/libgpuos_cuda.so
TAG=nobatch-mixed timeout 60 python tools/probe/c2.py
TAG=nobatch-contig GB_FORCE_OP=0 GB_FORCE_LAYOUT=0 GB_FORCE_DT=0 timeout 60 python tools/probe/c2.py
timeout 30 ./build/probe/profile_worker 10000 4096 2 | tail -2 | head -1
