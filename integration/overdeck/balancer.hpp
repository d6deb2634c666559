#pragma once
// Drop-in replacement of the reference's overdeck/balancer.hpp
// (/root/reference/proj/include/overdeck/balancer.hpp:1-184): the same public
// names, types and signatures, served by libod_b200 through its C ABI
// (include/overdeck_b200.h).  Put this directory ahead of the reference's
// include directory (-I integration -I .../proj/include) and every caller --
// Engine::run_epoch (engine.hpp:252-268), the CLI, the tests -- runs the B200
// build's balancers without a source change.  oracle/Makefile builds the
// reference's own acceptance suite against it (oracle/_ref/acceptance_b200;
// tests/test_dropin_acceptance.py).
//
//   BalancePolicy        balancer.hpp:15-27   (plain value type, same fields)
//   should_balance       balancer.hpp:29-32   -> od_should_balance
//   greedy_lb            balancer.hpp:36-63   -> od_greedy_lb
//   refine_swap_lb       balancer.hpp:68-152  -> od_refine_swap_lb
//   plan_cost            balancer.hpp:157-175 -> od_plan_cost
//   plan_to_json         balancer.hpp:177-182 (rendering only)
#include <cstdint>
#include <string>
#include <vector>

#include "json.hpp"
#include "overdeck/cluster.hpp"
#include "overdeck/gpu_cost.hpp"
#include "overdeck_b200.h"

namespace overdeck {

namespace b200 {
// C ABI return codes back to the reference's exception types (main.cpp:17-19)
inline void check(int rc) {
  if (rc == OD_OK) return;
  const std::string msg = od_last_error();
  if (rc == OD_EVALIDATION) throw ValidationError(msg);
  throw RuntimeFault(msg);
}
inline std::vector<int32_t> assignment(const Mapping& m) {
  std::vector<int32_t> a(static_cast<size_t>(m.vp_count()));
  for (VpId v = 0; v < m.vp_count(); ++v) a[static_cast<size_t>(v)] = m.proc_of(v);
  return a;
}
inline MigrationPlan plan_of(const std::vector<od_move>& out, int32_t n, Strategy s) {
  MigrationPlan p;
  p.strategy = s;
  p.moves.reserve(static_cast<size_t>(n));
  for (int32_t i = 0; i < n; ++i) p.moves.push_back(Move{out[i].vp, out[i].from, out[i].to});
  return p;
}
}  // namespace b200

struct BalancePolicy {
  Strategy first_call_strategy = Strategy::Greedy;
  Strategy later_call_strategy = Strategy::RefineSwap;
  double trigger_threshold = 1.0;
  double refine_tolerance = 0.02;

  void validate() const {
    if (trigger_threshold < 1.0) throw ValidationError("policy.trigger_threshold must be >= 1");
    if (refine_tolerance < 0.0) throw ValidationError("policy.refine_tolerance must be >= 0");
  }
};

inline bool should_balance(const std::vector<double>& proc_totals, const BalancePolicy& policy) {
  int32_t out = 0;
  b200::check(od_should_balance(proc_totals.data(), static_cast<int32_t>(proc_totals.size()),
                                policy.trigger_threshold, &out));
  return out != 0;
}

inline MigrationPlan greedy_lb(const LoadVector& loads, const Mapping& mapping) {
  const std::vector<int32_t> a = b200::assignment(mapping);
  std::vector<od_move> out(a.size() + 1);
  int32_t n = 0;
  b200::check(od_greedy_lb(loads.data(), static_cast<int32_t>(loads.size()), a.data(),
                           mapping.vp_count(), mapping.proc_count(), out.data(),
                           static_cast<int32_t>(out.size()), &n));
  return b200::plan_of(out, n, Strategy::Greedy);
}

inline MigrationPlan refine_swap_lb(const LoadVector& loads, const Mapping& mapping,
                                    double tolerance = 0.02) {
  const std::vector<int32_t> a = b200::assignment(mapping);
  // at most K*P rounds of at most two moves each
  std::vector<od_move> out(2 * a.size() * static_cast<size_t>(mapping.proc_count()) + 1);
  int32_t n = 0;
  b200::check(od_refine_swap_lb(loads.data(), static_cast<int32_t>(loads.size()), a.data(),
                                mapping.vp_count(), mapping.proc_count(), tolerance, out.data(),
                                static_cast<int32_t>(out.size()), &n));
  return b200::plan_of(out, n, Strategy::RefineSwap);
}

inline double plan_cost(const MigrationPlan& plan, const std::vector<VirtualProcess>& vps,
                        const ClusterState& cluster, const GpuModel& gpu) {
  std::vector<od_move> mv;
  mv.reserve(plan.moves.size());
  for (const Move& m : plan.moves) mv.push_back(od_move{m.vp, m.from, m.to});
  std::vector<int64_t> bytes;
  bytes.reserve(vps.size());
  for (const VirtualProcess& v : vps) bytes.push_back(v.data_bytes);
  const od_gpu_model g{gpu.launch_overhead, gpu.per_item_time, gpu.saturation_floor,
                       gpu.h2d_bandwidth, gpu.d2h_bandwidth, gpu.async_overlap_gain};
  double out = 0.0;
  b200::check(od_plan_cost(mv.data(), static_cast<int32_t>(mv.size()), bytes.data(),
                           static_cast<int32_t>(bytes.size()), cluster.spec.procs_per_node,
                           cluster.spec.nodes, cluster.spec.network_bandwidth,
                           cluster.spec.network_latency, &g, &out));
  return out;
}

inline nlohmann::json plan_to_json(const MigrationPlan& plan) {
  nlohmann::json moves = nlohmann::json::array();
  for (const Move& m : plan.moves) moves.push_back({{"vp", m.vp}, {"from", m.from}, {"to", m.to}});
  return {{"strategy", to_string(plan.strategy)}, {"moves", moves}};
}

}  // namespace overdeck
