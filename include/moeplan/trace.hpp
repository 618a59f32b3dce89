// B200 FSEP framework -- routing traces.  Two halves: the synthetic drifting-skew
// generator, and the JSONL record format ({"iter","layer","R"} per line) shared with
// the reference (/root/reference/proj/include/moeplan/trace.hpp:32-64).  The GPU
// runtime exports what it observes in the same format (mp_fsep_layer_histogram ->
// mp_trace), so reference tooling can replay real B200 routing.
#pragma once
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "moeplan/types.hpp"

namespace moeplan {

// ---------------------------------------------------------------- generation

// Dirichlet-like popularity per layer (skew_alpha), drifting by a Gaussian step of
// drift_sigma per iteration; every device routes tokens_per_device token-slots.
struct TraceGenSpec {
  int n_devices = 0, n_experts = 0;
  int n_layers = 1, n_iterations = 1;
  TokenCount tokens_per_device = 0;
  double skew_alpha = 1.0, drift_sigma = 0.0;
  std::uint64_t seed = 0;
};

// Records ordered by (iteration, layer).
std::vector<TraceRecord> generate_trace(const TraceGenSpec& spec);

// The popularity generate_trace rounds into its R rows, out[layer][iter][expert]; the
// GPU bench turns it into the Gumbel-top-k routing bias of the drifting config.
std::vector<std::vector<std::vector<double>>> trace_popularity(const TraceGenSpec& spec);

// ---------------------------------------------------------------- JSONL I/O

std::vector<TraceRecord> parse_trace(std::istream& in);
void write_trace(const std::vector<TraceRecord>& records, std::ostream& out);
// file variants of the two above
std::vector<TraceRecord> load_trace(const std::string& path);
void save_trace(const std::vector<TraceRecord>& records, const std::string& path);

// ---------------------------------------------------------------- statistics

// Per-record expert loads and shares of the record's token total.
struct TraceStats {
  std::uint32_t iteration = 0, layer = 0;
  TokenCount total_tokens = 0;
  bool zero_total = false;  // no tokens: every share is 1/E
  std::vector<TokenCount> expert_load;
  std::vector<double> expert_share;
  double max_share = 0.0, min_share = 0.0;
};

std::vector<TraceStats> trace_stats(const std::vector<TraceRecord>& records);

}  // namespace moeplan
