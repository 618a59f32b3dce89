// B200 FSEP framework -- host load-balancing planner (the "Planner" stage of the
// FSEP layer step).  Same API and bit-exact semantics as the reference planner
// (/root/reference/proj/include/moeplan/planner.hpp:32-100,
//  /root/reference/proj/src/planner.cpp:52-414); implementation is independent
// (see paper_2602_11686_b200/csrc/host/planner.cpp).  All functions are pure and
// re-entrant, so the runtime calls them from a host worker thread while the GPU
// streams run the previous step.
#pragma once
#include <cstdint>
#include <span>
#include <vector>

#include "moeplan/cost.hpp"
#include "moeplan/rng.hpp"
#include "moeplan/topology.hpp"
#include "moeplan/types.hpp"

namespace moeplan {

ReplicaVector replica_allocation(std::span<const double> expert_loads, int n_devices, int n_experts,
                                 int capacity);

ExpertLayout expert_relocation(const ReplicaVector& replicas, std::span<const double> expert_loads,
                               const Topology& topology, int capacity);

ReplicaVector perturb_replicas(const ReplicaVector& replicas, int n_devices, Rng& rng);

RoutingPlan lite_routing(const RoutingMatrix& routing, const ExpertLayout& layout, const Topology& topology);

ExpertLayout static_ep_layout(int n_devices, int n_experts, int capacity);

ExpertLayout even_replication_layout(const Topology& topology, int n_experts, int capacity);

enum class HistoryMode { last, ema };

struct LayoutSearchSpec {
  int epsilon = 2;
  std::uint64_t seed = 0;
  HistoryMode history_mode = HistoryMode::last;
  double ema_decay = 0.5;
};

struct AggregatedRouting {
  int n_devices = 0;
  int n_experts = 0;
  std::vector<double> weights;
  double at(int device, int expert) const {
    return weights[static_cast<std::size_t>(device) * n_experts + expert];
  }
  std::vector<double> expert_loads() const;
  RoutingMatrix rounded() const;
};

AggregatedRouting aggregate_history(std::span<const RoutingMatrix> history, HistoryMode mode, double ema_decay);

ExpertLayout plan_layout(std::span<const RoutingMatrix> history, const Topology& topology,
                         const CostParams& params, int capacity, const LayoutSearchSpec& spec);

}  // namespace moeplan
