// Golden workload checksums from the reference itself (TEST INFRASTRUCTURE
// ONLY).  Compiled against /root/reference/proj/include by oracle/Makefile;
// run here (the container) by tests/golden/make_bench_checksums.sh, output
// committed as tests/golden/bench_checksums.json.
//
// For each of the five reference bench workloads (bench.hpp:290-957) and
// seeds 1..5 at the acceptance C10 sizes (acceptance_main.cpp:909-940), it runs
// the reference's Baseline mode (every operator on the reference's CPU
// kernels) and prints the FNV-1a output checksum per row.  The GPU gates
// (tools/bench/gpuos_gates.cpp) rebuild the same workloads with the same
// seeds and compare.
#include <gpuos/bench.hpp>

#include <cstdio>

using namespace gpuos;

int main() {
  std::printf("{\n  \"source\": \"reference run_bench, BenchMode::Baseline (CPU kernels), acceptance C10 specs\",\n");
  std::printf("  \"rows\": [\n");
  bool first = true;
  for (uint64_t seed = 1; seed <= 5; ++seed) {
    for (const BenchWorkload w : {BenchWorkload::Elementwise, BenchWorkload::Attention, BenchWorkload::Mixed,
                                  BenchWorkload::Injection, BenchWorkload::Contention}) {
      BenchSpec spec;
      spec.workload = w;
      spec.seed = seed;
      spec.workers = 2;
      spec.mode = BenchMode::Baseline;
      spec.elems = {1024};
      spec.submitters = {1, 2};
      switch (w) {  // acceptance_main.cpp:917-923
        case BenchWorkload::Elementwise: spec.ops = 20; spec.reps = 5; break;
        case BenchWorkload::Attention: spec.ops = 8; spec.reps = 1; break;
        case BenchWorkload::Mixed: spec.ops = 30; spec.reps = 1; break;
        case BenchWorkload::Injection: spec.ops = 40; spec.reps = 5; break;
        case BenchWorkload::Contention: spec.ops = 40; spec.reps = 5; break;
      }
      const BenchReport rep = run_bench(spec);
      for (const BenchRow& r : rep.rows) {
        std::printf("%s    {\"workload\": \"%s\", \"seed\": %llu, \"config\": %llu, \"aux\": %llu, \"checksum\": \"%016llx\"}",
                    first ? "" : ",\n", r.workload.c_str(), (unsigned long long)seed, (unsigned long long)r.config,
                    (unsigned long long)(r.workload == "mixed" ? r.aux : 0), (unsigned long long)r.checksum);
        first = false;
      }
    }
  }
  std::printf("\n  ]\n}\n");
  return 0;
}
