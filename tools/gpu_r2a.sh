cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
echo "== smoke"; timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "== smoke under ncu launch list"; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu.log 2>&1; echo "rc $?"; tail -2 gpurun_out/smoke_ncu.log; grep -c worker gpurun_out/smoke_launches.csv
echo "== submit cost"; timeout 120 ./build/probe/submit_cost 2>&1 | tail -8
echo "== cpp"; timeout 300 stdbuf -oL ./build/cpp/test_runtime > gpurun_out/cpp.log 2>&1; echo rc $?; tail -1 gpurun_out/cpp.log
