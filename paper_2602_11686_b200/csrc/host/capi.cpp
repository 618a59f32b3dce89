// C ABI of the host planner: the reference's mp_* surface
// (/root/reference/proj/include/moeplan.h:46-107) plus the array-level
// mp_fsep_* planner entry points declared in include/moeplan_fsep.h.
#include <algorithm>
#include <limits>
#include <memory>
#include <vector>

#include "capi_common.hpp"
#include "moeplan/commands.hpp"
#include "moeplan/config.hpp"
#include "moeplan/planner.hpp"
#include "moeplan_fsep.h"

using namespace moeplan;
using moeplan::capi::dup_string;
using moeplan::capi::guarded;
using moeplan::capi::require;

extern "C" {
struct mp_trace {
  std::vector<TraceRecord> records;
  std::vector<std::uint32_t> layers;
  std::uint32_t n_devices = 0, n_experts = 0;  // for traces built by mp_fsep_trace_append
};
struct mp_config {
  RunConfig cfg;
};
struct mp_fsep_planner {
  RunConfig cfg;
  Topology topo;
  LayoutSearchSpec spec;
  std::vector<RoutingMatrix> history;
  int n_devices;
};
}

namespace moeplan::capi {
std::string& last_error() {
  thread_local std::string text;
  return text;
}
}  // namespace moeplan::capi

namespace {
mp_trace* make_trace(std::vector<TraceRecord> recs) {
  auto* t = new mp_trace{std::move(recs), {}};
  t->layers = distinct_layers(t->records);
  return t;
}

RoutingMatrix matrix_from(const uint64_t* R, uint32_t n, uint32_t e) {
  RoutingMatrix m(static_cast<int>(n), static_cast<int>(e));
  std::copy(R, R + static_cast<std::size_t>(n) * e, m.data());
  return m;
}

ExpertLayout layout_from(const uint8_t* A, uint32_t n, uint32_t e) {
  ExpertLayout l(static_cast<int>(e), static_cast<int>(n));
  for (uint32_t j = 0; j < e; ++j)
    for (uint32_t d = 0; d < n; ++d)
      if (A[static_cast<std::size_t>(j) * n + d]) l.place(static_cast<int>(j), static_cast<int>(d));
  return l;
}

void layout_to(const ExpertLayout& l, uint8_t* A) {
  for (int j = 0; j < l.n_experts(); ++j)
    for (int d = 0; d < l.n_devices(); ++d) A[static_cast<std::size_t>(j) * l.n_devices() + d] = l.hosts(j, d);
}
}  // namespace

extern "C" {

const char* mp_status_name(mp_status s) {
  switch (s) {
    case MP_OK: return "ok";
    case MP_ERR_INVALID_ARGUMENT: return "invalid_argument";
    case MP_ERR_PARSE: return "parse";
    case MP_ERR_IO: return "io";
    case MP_ERR_INFEASIBLE: return "infeasible";
    case MP_ERR_BUDGET_EXCEEDED: return "budget_exceeded";
    case MP_ERR_INTERNAL: return "internal";
    case MP_ERR_DEVICE: return "device";
  }
  return "unknown";
}

const char* mp_last_error(void) { return moeplan::capi::last_error().c_str(); }

void mp_string_free(char* text) { std::free(text); }

mp_status mp_trace_generate(const char* spec_json, const uint64_t* seed_override, mp_trace** out) {
  return guarded([&] {
    require(spec_json && out, "mp_trace_generate: NULL argument");
    TraceGenSpec spec = parse_gen_spec(spec_json, seed_override == nullptr);
    if (seed_override) spec.seed = *seed_override;
    *out = make_trace(generate_trace(spec));
  });
}

mp_status mp_trace_load(const char* path, mp_trace** out) {
  return guarded([&] {
    require(path && out, "mp_trace_load: NULL argument");
    *out = make_trace(load_trace(path));
  });
}

mp_status mp_trace_save(const mp_trace* trace, const char* path) {
  return guarded([&] {
    require(trace && path, "mp_trace_save: NULL argument");
    save_trace(trace->records, path);
  });
}

mp_status mp_trace_dims(const mp_trace* trace, uint32_t* n_devices, uint32_t* n_experts, uint32_t* n_records) {
  return guarded([&] {
    require(trace, "mp_trace_dims: NULL trace");
    const bool any = !trace->records.empty();
    if (n_devices) *n_devices = any ? static_cast<uint32_t>(trace->records.front().routing.n_devices()) : 0;
    if (n_experts) *n_experts = any ? static_cast<uint32_t>(trace->records.front().routing.n_experts()) : 0;
    if (n_records) *n_records = static_cast<uint32_t>(trace->records.size());
  });
}

mp_status mp_trace_layer_count(const mp_trace* trace, uint32_t* count) {
  return guarded([&] {
    require(trace && count, "mp_trace_layer_count: NULL argument");
    *count = static_cast<uint32_t>(trace->layers.size());
  });
}

mp_status mp_trace_layer_at(const mp_trace* trace, uint32_t index, uint32_t* layer) {
  return guarded([&] {
    require(trace && layer, "mp_trace_layer_at: NULL argument");
    require(index < trace->layers.size(), "mp_trace_layer_at: index out of range");
    *layer = trace->layers[index];
  });
}

mp_status mp_trace_stats_json(const mp_trace* trace, char** out_json) {
  return guarded([&] {
    require(trace && out_json, "mp_trace_stats_json: NULL argument");
    *out_json = dup_string(stats_json(trace->records));
  });
}

void mp_trace_free(mp_trace* trace) { delete trace; }

mp_status mp_config_parse(const char* config_json, mp_config** out) {
  return guarded([&] {
    require(config_json && out, "mp_config_parse: NULL argument");
    *out = new mp_config{parse_run_config(config_json)};
  });
}

mp_status mp_config_load(const char* path, mp_config** out) {
  return guarded([&] {
    require(path && out, "mp_config_load: NULL argument");
    *out = new mp_config{load_run_config(path)};
  });
}

mp_status mp_config_set_seed(mp_config* config, uint64_t seed) {
  return guarded([&] {
    require(config, "mp_config_set_seed: NULL config");
    config->cfg.search.seed = seed;
    config->cfg.has_seed = true;
  });
}

const char* mp_config_trace_path(const mp_config* config) { return config ? config->cfg.trace_path.c_str() : ""; }
const char* mp_config_out_path(const mp_config* config) { return config ? config->cfg.out_path.c_str() : ""; }
void mp_config_free(mp_config* config) { delete config; }

mp_status mp_plan_layer_json(const mp_config* config, const mp_trace* trace, uint32_t layer, char** out_json) {
  return guarded([&] {
    require(config && trace && out_json, "mp_plan_layer_json: NULL argument");
    *out_json = dup_string(plan_layer_json(config->cfg, trace->records, layer));
  });
}

mp_status mp_simulate(const mp_config* config, const mp_trace* trace, const char* schedulers_csv,
                      char** out_report_json, char** out_series_csv) {
  return guarded([&] {
    require(config && trace && schedulers_csv, "mp_simulate: NULL argument");
    auto [report, csv] = simulate_artifacts(config->cfg, trace->records, parse_scheduler_list(schedulers_csv));
    if (out_report_json) *out_report_json = dup_string(report);
    if (out_series_csv) *out_series_csv = dup_string(csv);
  });
}

mp_status mp_analyze_json(const mp_config* config, char** out_json) {
  return guarded([&] {
    require(config && out_json, "mp_analyze_json: NULL argument");
    *out_json = dup_string(analyze_json(config->cfg));
  });
}

mp_status mp_oracle_gap_json(const mp_config* config, const char* instance_json, char** out_json) {
  return guarded([&] {
    require(config && instance_json && out_json, "mp_oracle_gap_json: NULL argument");
    *out_json = dup_string(oracle_gap_json(config->cfg, parse_instance(instance_json)));
  });
}

/* ---------------------------- array-level planner ------------------------ */

mp_status mp_fsep_planner_create(const mp_config* config, uint32_t n_devices, uint32_t layer,
                                 mp_fsep_planner** out) {
  return guarded([&] {
    require(config && out, "mp_fsep_planner_create: NULL argument");
    const RunConfig& c = config->cfg;
    const Topology& topo = c.require_topology();
    c.require_cost();
    c.require_model();
    c.require_seed();
    require(topo.n_devices() == static_cast<int>(n_devices), "mp_fsep_planner_create: topology size != n_devices");
    LayoutSearchSpec spec = c.search;
    spec.seed = mix_seed(c.search.seed, 0x6c617972, layer);
    *out = new mp_fsep_planner{c, topo, spec, {}, static_cast<int>(n_devices)};
  });
}

mp_status mp_fsep_planner_observe(mp_fsep_planner* p, const uint64_t* R) {
  return guarded([&] {
    require(p && R, "mp_fsep_planner_observe: NULL argument");
    p->history.push_back(matrix_from(R, static_cast<uint32_t>(p->n_devices), static_cast<uint32_t>(p->cfg.n_experts)));
  });
}

mp_status mp_fsep_planner_next(mp_fsep_planner* p, uint8_t* A_out) {
  return guarded([&] {
    require(p && A_out, "mp_fsep_planner_next: NULL argument");
    const ExpertLayout l = p->history.empty()
                               ? even_replication_layout(p->topo, p->cfg.n_experts, p->cfg.capacity)
                               : plan_layout(p->history, p->topo, *p->cfg.cost, p->cfg.capacity, p->spec);
    layout_to(l, A_out);
  });
}

void mp_fsep_planner_free(mp_fsep_planner* p) { delete p; }

mp_status mp_fsep_plan_next(const mp_config* config, const uint64_t* R, uint32_t n_devices, uint32_t layer,
                            uint8_t* A_out) {
  return guarded([&] {
    require(config && R && A_out, "mp_fsep_plan_next: NULL argument");
    const RunConfig& c = config->cfg;
    const Topology& topo = c.require_topology();
    const CostParams& params = c.require_cost();
    c.require_model();
    c.require_seed();
    require(topo.n_devices() == static_cast<int>(n_devices), "mp_fsep_plan_next: topology size != n_devices");
    LayoutSearchSpec spec = c.search;
    spec.seed = mix_seed(c.search.seed, 0x6c617972, layer);  // per-layer seed, as mp_plan_layer_json
    const std::vector<RoutingMatrix> hist{matrix_from(R, n_devices, static_cast<uint32_t>(c.n_experts))};
    layout_to(plan_layout(hist, topo, params, c.capacity, spec), A_out);
  });
}

mp_status mp_fsep_plan_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, double bandwidth,
                              double v_comm, double v_comp, double b_comp, uint32_t epsilon, uint64_t seed,
                              const uint64_t* R, uint8_t* A_out) {
  return guarded([&] {
    require(R && A_out, "mp_fsep_plan_layout: NULL argument");
    const Topology topo(1, static_cast<int>(n_devices), bandwidth, bandwidth);
    LayoutSearchSpec spec;
    spec.epsilon = static_cast<int>(epsilon);
    spec.seed = seed;
    const std::vector<RoutingMatrix> hist{matrix_from(R, n_devices, n_experts)};
    layout_to(plan_layout(hist, topo, CostParams{v_comm, v_comp, b_comp, 0}, static_cast<int>(capacity), spec), A_out);
  });
}

mp_status mp_fsep_lite_routing(uint32_t n_devices, uint32_t n_experts, const uint64_t* R, const uint8_t* A,
                               uint64_t* S_out) {
  return guarded([&] {
    require(R && A && S_out, "mp_fsep_lite_routing: NULL argument");
    const Topology topo(1, static_cast<int>(n_devices), 1.0, 1.0);
    const RoutingPlan plan =
        lite_routing(matrix_from(R, n_devices, n_experts), layout_from(A, n_devices, n_experts), topo);
    std::fill(S_out, S_out + static_cast<std::size_t>(n_devices) * n_experts * n_devices, 0);
    for (const PlanEntry& e : plan.entries)
      S_out[(static_cast<std::size_t>(e.src) * n_experts + e.expert) * n_devices + e.dst] = e.tokens;
  });
}

mp_status mp_fsep_static_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, uint8_t* A_out) {
  return guarded([&] {
    require(A_out, "mp_fsep_static_layout: NULL argument");
    layout_to(static_ep_layout(static_cast<int>(n_devices), static_cast<int>(n_experts), static_cast<int>(capacity)),
              A_out);
  });
}

mp_status mp_fsep_even_layout(uint32_t n_devices, uint32_t n_experts, uint32_t capacity, uint8_t* A_out) {
  return guarded([&] {
    require(A_out, "mp_fsep_even_layout: NULL argument");
    const Topology topo(1, static_cast<int>(n_devices), 1.0, 1.0);
    layout_to(even_replication_layout(topo, static_cast<int>(n_experts), static_cast<int>(capacity)), A_out);
  });
}

mp_status mp_fsep_trace_create(uint32_t n_devices, uint32_t n_experts, mp_trace** out) {
  return guarded([&] {
    require(out && n_devices > 0 && n_experts > 0, "mp_fsep_trace_create: bad argument");
    auto* t = make_trace({});
    t->n_devices = n_devices;
    t->n_experts = n_experts;
    *out = t;
  });
}

mp_status mp_fsep_trace_append(mp_trace* trace, uint32_t iteration, uint32_t layer, const uint64_t* R) {
  return guarded([&] {
    require(trace && R, "mp_fsep_trace_append: NULL argument");
    uint32_t n = trace->n_devices, e = trace->n_experts;
    if (!trace->records.empty()) {
      n = static_cast<uint32_t>(trace->records.front().routing.n_devices());
      e = static_cast<uint32_t>(trace->records.front().routing.n_experts());
    }
    require(n > 0 && e > 0, "mp_fsep_trace_append: trace has no dimensions (use mp_fsep_trace_create)");
    for (const TraceRecord& r : trace->records)
      require(!(r.iteration == iteration && r.layer == layer), "mp_fsep_trace_append: duplicate (iter, layer) pair");
    TraceRecord rec;
    rec.iteration = iteration;
    rec.layer = layer;
    rec.routing = matrix_from(R, n, e);
    trace->records.push_back(std::move(rec));
    std::sort(trace->records.begin(), trace->records.end(), [](const TraceRecord& a, const TraceRecord& b) {
      return a.iteration != b.iteration ? a.iteration < b.iteration : a.layer < b.layer;
    });
    trace->layers = distinct_layers(trace->records);
  });
}

mp_status mp_fsep_trace_popularity(const char* spec_json, double* out, uint64_t capacity) {
  return guarded([&] {
    require(spec_json && out, "mp_fsep_trace_popularity: NULL argument");
    const TraceGenSpec spec = parse_gen_spec(spec_json, true);
    const auto pop = trace_popularity(spec);
    const uint64_t need = static_cast<uint64_t>(spec.n_layers) * spec.n_iterations * spec.n_experts;
    require(capacity >= need, "mp_fsep_trace_popularity: output too small");
    uint64_t k = 0;
    for (const auto& layer : pop)
      for (const auto& it : layer)
        for (double v : it) out[k++] = v;
  });
}

mp_status mp_fsep_time_cost(uint32_t n_devices, uint32_t n_experts, const uint64_t* R, const uint8_t* A,
                            double bandwidth, double v_comm, double v_comp, double b_comp, double* t_comm,
                            double* t_comp, double* t_total, uint64_t* max_recv) {
  return guarded([&] {
    require(R && A, "mp_fsep_time_cost: NULL argument");
    const Topology topo(1, static_cast<int>(n_devices), bandwidth, bandwidth);
    const CostBreakdown cb = time_cost(
        lite_routing(matrix_from(R, n_devices, n_experts), layout_from(A, n_devices, n_experts), topo), topo,
        CostParams{v_comm, v_comp, b_comp, 0});
    if (t_comm) *t_comm = cb.t_comm;
    if (t_comp) *t_comp = cb.t_comp;
    if (t_total) *t_total = cb.t_total;
    if (max_recv) *max_recv = cb.max_recv_tokens();
  });
}

}  // extern "C"
