// B200 FSEP framework -- command-level entry points behind the C ABI
// (/root/reference/proj/include/moeplan/commands.hpp:30-54).
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "moeplan/config.hpp"
#include "moeplan/sim.hpp"

namespace moeplan {

std::vector<std::uint32_t> distinct_layers(const std::vector<TraceRecord>& records);
std::string plan_layer_json(const RunConfig& config, const std::vector<TraceRecord>& trace, std::uint32_t layer);
std::pair<std::string, std::string> simulate_artifacts(const RunConfig& config,
                                                       const std::vector<TraceRecord>& trace,
                                                       const std::vector<SchedulerKind>& schedulers);
std::vector<SchedulerKind> parse_scheduler_list(const std::string& csv);
std::string analyze_json(const RunConfig& config);
std::string stats_json(const std::vector<TraceRecord>& trace);
// Greedy planner vs the exact optimum on one tiny instance (mp_oracle_gap_json).
std::string oracle_gap_json(const RunConfig& config, const RoutingMatrix& instance);

}  // namespace moeplan
