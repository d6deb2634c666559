// TEST INFRASTRUCTURE: prints the reference simulator's JSON report
// (report.hpp:69-114) of every preset plus randomised configurations, so the
// same source compiled against the reference's balancer/measurement headers and
// against integration/overdeck/ (libod_b200 behind the C ABI) can be diffed
// byte for byte (oracle/Makefile: _ref/presets_ref, _ref/presets_b200).
#include <cstdio>
#include <random>

#include "overdeck/config.hpp"
#include "overdeck/presets.hpp"
#include "overdeck/report.hpp"

using namespace overdeck;

int main() {
  ExperimentConfig cfgs[] = {preset_exp_a(), preset_exp_a_baseline_p2(), preset_exp_b(),
                             preset_exp_c()};
  for (const ExperimentConfig& c : cfgs)
    std::printf("%s\n", render_report(run_experiment(c), ReportFormat::Json).c_str());
  // random shapes: processors, VP counts, thresholds, noise and strategies
  std::mt19937_64 rng(20261019);
  for (int i = 0; i < 40; ++i) {
    ExperimentConfig c = preset_exp_c();
    c.cluster.nodes = 1 + int(rng() % 4);
    c.cluster.procs_per_node = 1 + int(rng() % 3);
    const int P = c.cluster.nodes * c.cluster.procs_per_node;
    c.decomposition.ky = P + int(rng() % 24);
    c.policy.trigger_threshold = 1.0 + double(rng() % 10) / 100.0;
    c.policy.first_call_strategy = rng() % 2 ? Strategy::Greedy : Strategy::RefineSwap;
    c.policy.later_call_strategy = rng() % 2 ? Strategy::Greedy : Strategy::RefineSwap;
    c.seed = rng();
    c.epochs = 2 + int(rng() % 4);
    std::printf("%s\n", render_report(run_experiment(c), ReportFormat::Json).c_str());
  }
  return 0;
}
