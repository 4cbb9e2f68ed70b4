// serialize.hpp -- artifact formats of the reference's serialize module
// (serialize.hpp:18-36): plans (declared in planner.hpp), reconfiguration
// action lists and SimReport tables, byte-compatible with the reference.
#pragma once

#include <string>
#include <string_view>

#include "moeb200/planner.hpp"
#include "moeb200/reconfig.hpp"
#include "moeb200/simulator.hpp"

namespace moeb200 {

// moeserve.reconfig.v1 (serialize.cpp:160-206): read recomputes the cost at
// `hw` and rejects a stored bytes_moved that disagrees with the actions.
std::string write_reconfig(const ReconfigPlan& plan, const ModelProfile& profile);
ReconfigPlan read_reconfig(std::string_view document, const ModelProfile& profile, const HardwareProfile& hw);

// SimReport as a one-row CSV table / a JSON object (serialize.cpp:218-243).
std::string report_csv(const SimReport& report);
std::string report_json(const SimReport& report);

// A double as nlohmann/json 3.11.3 dumps it.
std::string json_double(double v);

}  // namespace moeb200
