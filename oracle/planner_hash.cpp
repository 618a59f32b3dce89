// Test infrastructure only (never shipped): a hash of the planner's outputs over a
// seeded stream of random instances, written against the moeplan C++ API alone
// (planner.hpp / cost.hpp / types.hpp / topology.hpp), so the SAME source compiles
// against the reference library (/root/reference/proj, linked by oracle/build_ref.sh)
// and against this build (include/ + libmoeplan_b200.so).  Equal hashes = the two
// planners agree bit for bit on every instance: plan_layout (history 1-3 steps,
// last / EMA, epsilon 2-5), lite_routing entries and the time_cost doubles.
// SURVEY §7 step 2 ("a 20k-random-instance hash-equality test").
//
// usage: planner_hash COUNT SEED   ->   prints "<count> <hash>"
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "moeplan/cost.hpp"
#include "moeplan/planner.hpp"
#include "moeplan/topology.hpp"
#include "moeplan/types.hpp"

namespace {

struct Fnv {
  std::uint64_t h = 1469598103934665603ull;
  void bytes(const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  }
  void u64(std::uint64_t v) { bytes(&v, sizeof(v)); }
  void f64(double v) {
    std::uint64_t b;
    std::memcpy(&b, &v, sizeof(b));
    u64(b);
  }
};

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s COUNT SEED\n", argv[0]);
    return 2;
  }
  const long count = std::atol(argv[1]);
  std::mt19937_64 g(std::strtoull(argv[2], nullptr, 10));
  auto pick = [&](std::uint64_t n) { return static_cast<int>(g() % n); };
  Fnv f;
  long done = 0;
  for (long i = 0; i < count; ++i) {
    const int nodes = 1 + pick(4), dpn = 1 + pick(8), n = nodes * dpn;
    const int c = 1 + pick(4);
    const int e_max = n * c < 64 ? n * c : 64;
    const int e = c + pick(static_cast<std::uint64_t>(e_max - c + 1));
    const double b_intra = 1e9 * (1 + pick(900)), b_inter = 1e8 * (1 + pick(900));
    const moeplan::Topology topo(nodes, dpn, b_intra, b_inter);
    const moeplan::CostParams params{512.0 * (1 + pick(16)), 1e6 * (1 + pick(400)), 1e12 * (1 + pick(2000)),
                                     pick(2)};
    moeplan::LayoutSearchSpec spec;
    spec.epsilon = 2 + pick(4);
    spec.seed = g();
    spec.history_mode = pick(2) ? moeplan::HistoryMode::ema : moeplan::HistoryMode::last;
    spec.ema_decay = 0.1 * (1 + pick(9));
    // skewed token counts: a hot subset of experts, zero cells, occasional idle devices
    std::vector<moeplan::RoutingMatrix> history;
    const int steps = 1 + pick(3);
    for (int s = 0; s < steps; ++s) {
      moeplan::RoutingMatrix r(n, e);
      for (int d = 0; d < n; ++d) {
        const bool idle = pick(16) == 0;
        for (int j = 0; j < e; ++j) {
          const std::uint64_t base = static_cast<std::uint64_t>(pick(200));
          const bool hot = (static_cast<std::uint64_t>(j) * 2654435761u + s) % 5 == 0;
          r.at(d, j) = idle || pick(8) == 0 ? 0 : base * (hot ? 1 + pick(30) : 1);
        }
      }
      history.push_back(std::move(r));
    }
    const moeplan::ExpertLayout layout = moeplan::plan_layout(history, topo, params, c, spec);
    const moeplan::RoutingPlan plan = moeplan::lite_routing(history.back(), layout, topo);
    const moeplan::CostBreakdown cost = moeplan::time_cost(plan, topo, params);
    f.u64(static_cast<std::uint64_t>(n) << 32 | static_cast<std::uint64_t>(e));
    for (int j = 0; j < e; ++j)
      for (int d = 0; d < n; ++d) f.u64(layout.hosts(j, d) ? 1 : 0);
    for (const moeplan::PlanEntry& p : plan.entries) {
      f.u64(static_cast<std::uint64_t>(p.src) << 40 | static_cast<std::uint64_t>(p.expert) << 20 |
            static_cast<std::uint64_t>(p.dst));
      f.u64(p.tokens);
    }
    f.f64(cost.t_comm);
    f.f64(cost.t_comp);
    f.f64(cost.t_total);
    ++done;
  }
  std::printf("%ld %016llx\n", done, static_cast<unsigned long long>(f.h));
  return 0;
}
