// B200 FSEP framework -- deterministic text forms (%.9g doubles), byte-compatible
// with the reference serializers (/root/reference/proj/src/serialize.cpp:23-112).
#pragma once
#include <string>

#include "moeplan/sim.hpp"
#include "moeplan/types.hpp"

namespace moeplan {

std::string format_double(double value);
std::string layout_to_json(const ExpertLayout& layout, int capacity);
std::string plan_to_json(const RoutingPlan& plan, const RoutingMatrix& routing, const ExpertLayout& layout);
std::string report_to_json(const SimReport& report);
std::string report_to_csv(const SimReport& report);

}  // namespace moeplan
