// oracle/dropin/e2e_main.cpp — TEST-ONLY driver: the reference's experiment
// harness (run_experiment -> Simulator -> LocalScheduler x n + the global
// scheduler; harness.cpp, simulator.cpp:60-240, local_scheduler.cpp:165-266)
// on the experiment configurations of acceptance criteria 4-6
// (acceptance_main.cpp:216-366).  Linked once against the reference's own
// GlobalScheduler and once, through oracle/dropin/, against libe2sched.so
// (or the host emulation): the reports must be byte-identical.
//
//   e2e_main OUTDIR   writes OUTDIR/<name>.json and OUTDIR/<name>.csv, and one
//                     "name seconds requests" line per experiment on stdout
#include <chrono>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "kvsched/harness.hpp"

using namespace kvsched;

namespace {
ExperimentConfig experiment(const char* name, Archetype arch, PolicyName policy, uint64_t seed, double rps,
                            int64_t n, int64_t capacity, int batch, double decode_ms) {
  ExperimentConfig cfg;
  cfg.name = name;
  cfg.seed = seed;
  cfg.rps = rps;
  cfg.policy = policy;
  cfg.sim.n_gpus = 4;
  cfg.sim.scheduler.kv_capacity_tokens = capacity;
  cfg.sim.max_batch_requests = batch;
  cfg.sim.model.decode_per_token_ms = decode_ms;
  cfg.workload = WorkloadSpec::archetype_default(arch);
  cfg.workload.request_count = n;
  return cfg;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s OUTDIR\n", argv[0]);
    return 2;
  }
  const std::string out = argv[1];
  const std::vector<ExperimentConfig> cfgs = {
      // criterion 4 (conservation)
      experiment("c4_toolbench_e2full", Archetype::Toolbench, PolicyName::E2Full, 5, 11.0, 600, 20000, 8, 1.0),
      experiment("c4_docqa_rr", Archetype::DocQa, PolicyName::RoundRobin, 7, 5.0, 300, 200000, 8, 15.0),
      experiment("c4_embodied_nopd", Archetype::EmbodiedAgent, PolicyName::E2NoPdBalance, 9, 8.0, 500, 100000, 16,
                 2.0),
      // criterion 5 (determinism)
      experiment("c5_toolbench_lpf", Archetype::Toolbench, PolicyName::LongestPrefixFirstLocal, 3, 11.0, 500, 20000, 8,
                 1.0),
      // criterion 6 (ablation ordering), seed 1
      experiment("c6_full", Archetype::Toolbench, PolicyName::E2Full, 1, 11.0, 1500, 20000, 8, 1.0),
      experiment("c6_rr", Archetype::Toolbench, PolicyName::RoundRobin, 1, 11.0, 1500, 20000, 8, 1.0),
      experiment("c6_norebalance", Archetype::Toolbench, PolicyName::E2NoRebalance, 1, 11.0, 1500, 20000, 8, 1.0),
      experiment("c6_lpf", Archetype::Toolbench, PolicyName::LongestPrefixFirstLocal, 1, 11.0, 1500, 20000, 8, 1.0),
  };
  for (const ExperimentConfig& cfg : cfgs) {
    const auto t0 = std::chrono::steady_clock::now();
    const MetricsReport rep = run_experiment(cfg);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::ofstream(out + "/" + cfg.name + ".json") << rep.to_json().dump(2) << "\n";
    std::ofstream(out + "/" + cfg.name + ".csv") << rep.to_csv();
    std::printf("%s %.6f %lld\n", cfg.name.c_str(), s, (long long)rep.requests);
  }
  return 0;
}
