cd "${GRAFT_REPO_ROOT:-/root/repo}"
for e in 65536 16384 4096; do echo "bulk $e"; timeout 30 ./build/probe/profile_worker $((40960000/e)) $e 2 2>&1 | tail -2 | head -1; done
cp paper_2604_17861_b200/lib/libgpuos_cuda_nobulk.so paper_2604_17861_b200/lib/libgpuos_cuda.so
for e in 65536 16384 4096; do echo "nobulk $e"; timeout 30 ./build/probe/profile_worker $((40960000/e)) $e 2 2>&1 | tail -2 | head -1; done
