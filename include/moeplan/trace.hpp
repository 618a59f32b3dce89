// B200 FSEP framework -- routing traces: the synthetic drifting-skew generator and
// the JSONL record format {"iter","layer","R"} shared with the reference
// (/root/reference/proj/include/moeplan/trace.hpp:32-64).  The GPU runtime exports
// its observed histograms in the same format (mp_fsep_layer_histogram ->
// mp_trace), so reference tooling can replay real B200 routing.
#pragma once
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "moeplan/types.hpp"

namespace moeplan {

struct TraceGenSpec {
  int n_devices = 0;
  int n_experts = 0;
  int n_layers = 1;
  int n_iterations = 1;
  TokenCount tokens_per_device = 0;
  double skew_alpha = 1.0;
  double drift_sigma = 0.0;
  std::uint64_t seed = 0;
};

std::vector<TraceRecord> generate_trace(const TraceGenSpec& spec);

// Per-layer expert popularity (softmax of the drifting logits) for every iteration:
// out[layer][iter][expert].  This is the quantity generate_trace rounds into R rows;
// the GPU bench uses it as the Gumbel-top-k routing bias for the drifting config.
std::vector<std::vector<std::vector<double>>> trace_popularity(const TraceGenSpec& spec);

std::vector<TraceRecord> parse_trace(std::istream& in);
std::vector<TraceRecord> load_trace(const std::string& path);
void write_trace(const std::vector<TraceRecord>& records, std::ostream& out);
void save_trace(const std::vector<TraceRecord>& records, const std::string& path);

struct TraceStats {
  std::uint32_t iteration = 0;
  std::uint32_t layer = 0;
  TokenCount total_tokens = 0;
  std::vector<TokenCount> expert_load;
  std::vector<double> expert_share;
  double max_share = 0.0;
  double min_share = 0.0;
  bool zero_total = false;
};

std::vector<TraceStats> trace_stats(const std::vector<TraceRecord>& records);

}  // namespace moeplan
