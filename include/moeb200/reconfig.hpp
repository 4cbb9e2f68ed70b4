// reconfig.hpp -- plan-to-plan reconfiguration.
//
// Same semantics as the reference reconfig module (reconfig.hpp:12-58,
// reconfig.cpp:19-168): the minimal per-expert action list between two
// placements, with the releasing group (Offload, Quantize) ahead of the
// consuming group (Dequantize, Fetch), each in expert order; its CPU->GPU
// byte cost under the "16-bit master copy on the CPU" model; and a checked
// replay.  MoeEngine::reconfigure executes the list on the device.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "moeb200/planner.hpp"

namespace moeb200 {

enum class ActionKind { Offload, Fetch, Quantize, Dequantize };

struct ReconfigAction {
    ActionKind kind = ActionKind::Offload;
    ExpertId expert;
    Precision target_precision = Precision::P16;  // the expert's entry in the destination plan
    Location target_location = Location::CPU;
    friend constexpr bool operator==(const ReconfigAction&, const ReconfigAction&) = default;
};

struct ReconfigPlan {
    std::vector<ReconfigAction> actions;
    bytes_t bytes_moved = 0;      // CPU -> GPU bytes
    double est_downtime_s = 0.0;  // bytes_moved / transfer bandwidth
    uint64_t target_seed = 0;
    friend bool operator==(const ReconfigPlan&, const ReconfigPlan&) = default;
};

ReconfigPlan diff_plans(const PlacementPlan& from, const PlacementPlan& to, const ModelProfile& profile,
                        const HardwareProfile& hw);
// Replay with state checks; budget != null also checks the footprint from the
// first consuming action on and at the end.
PlacementPlan apply(const PlacementPlan& plan, const ReconfigPlan& actions, const ModelProfile& profile,
                    const HardwareProfile* budget = nullptr);
std::pair<bytes_t, double> estimate_cost(const ReconfigPlan& actions, const ModelProfile& profile,
                                         const HardwareProfile& hw);

}  // namespace moeb200
