#!/bin/bash
# Golden workload checksums from the reference itself: oracle/ref_bench_checksums.cpp
# (compiled against /root/reference by oracle/Makefile) runs the five reference bench
# workloads in Baseline mode (its CPU kernels), acceptance-C10 sizes, seeds 1..5.
set -e
cd "$(dirname "$0")/../.."
make -C oracle ref
./oracle/_ref/ref_bench_checksums > tests/golden/bench_checksums.json
