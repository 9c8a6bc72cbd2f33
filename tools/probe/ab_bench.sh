cd "${GRAFT_REPO_ROOT:-/root/repo}"
L=paper_2604_17861_b200/lib
cp $L/libgpuos_bench.so $L/libgpuos_bench_new.so
for i in 1 2 3; do
  for v in old new; do
    cp $L/libgpuos_bench_$v.so $L/libgpuos_bench.so
    timeout 200 python bench.py --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), round(d['host_submit_ns_per_task'],1))"
  done
done
cp $L/libgpuos_bench_new.so $L/libgpuos_bench.so
