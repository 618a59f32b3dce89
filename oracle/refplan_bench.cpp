// Test/benchmark infrastructure only (never shipped): times the UNMODIFIED
// reference planner hot path -- moeplan::plan_layout + moeplan::lite_routing,
// /root/reference/proj/src/planner.cpp:369-414 and :238-287 -- on one host
// core, exactly as run_simulation's inner loop calls it
// (/root/reference/proj/src/sim.cpp:114-148).  Linked against the reference
// objects by oracle/build_ref.sh.
//
// usage: refplan_bench N E C iters b_intra v_comm v_comp b_comp seed < R.txt
//   R.txt holds N*E unsigned counts (row-major, whitespace separated).
// prints one JSON line: per-call microseconds and the chosen layout.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <vector>

#include "moeplan/planner.hpp"

int main(int argc, char** argv) {
  if (argc < 10) {
    std::fprintf(stderr, "usage: %s N E C iters b_intra v_comm v_comp b_comp seed < R\n", argv[0]);
    return 2;
  }
  const int n = std::atoi(argv[1]), e = std::atoi(argv[2]), c = std::atoi(argv[3]);
  const int iters = std::atoi(argv[4]);
  const double bw = std::atof(argv[5]);
  moeplan::CostParams params{std::atof(argv[6]), std::atof(argv[7]), std::atof(argv[8]), 0};
  moeplan::LayoutSearchSpec spec;
  spec.seed = std::strtoull(argv[9], nullptr, 10);
  moeplan::RoutingMatrix r(n, e);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < e; ++j) std::cin >> r.at(i, j);
  moeplan::Topology topo(1, n, bw, bw);
  std::vector<moeplan::RoutingMatrix> history{r};
  moeplan::ExpertLayout layout;
  std::size_t entries = 0;
  auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it)
    layout = moeplan::plan_layout(history, topo, params, c, spec);
  auto t1 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; ++it)
    entries += moeplan::lite_routing(r, layout, topo).entries.size();
  auto t2 = std::chrono::steady_clock::now();
  double plan_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
  double route_us = std::chrono::duration<double, std::micro>(t2 - t1).count() / iters;
  std::printf("{\"plan_us\":%.3f,\"route_us\":%.3f,\"entries\":%zu,\"layout\":[", plan_us,
              route_us, entries / (iters > 0 ? iters : 1));
  for (int j = 0; j < e; ++j)
    for (int d = 0; d < n; ++d)
      std::printf("%s%d", (j | d) ? "," : "", layout.hosts(j, d) ? 1 : 0);
  std::printf("]}\n");
  return 0;
}
