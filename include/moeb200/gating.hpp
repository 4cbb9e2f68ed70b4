// gating.hpp -- routing records in the reference's trace contract.
//
// GatingTrace has the reference layout (gating.hpp:16-29): for every
// (token, layer) pair top_k distinct slots in ascending order at
// slots[(t*L + l)*k + i].  generate_trace is the reference's uniform router
// stand-in (gating.cpp:31-53); the engine's real K1 router exports its
// decisions in this same layout (MoeEngine::export_trace) so the counters of
// simulate() can be replayed on real routing.  Text format v1 as in
// gating.hpp:35-37.
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "moeb200/config.hpp"

namespace moeb200 {

struct GatingTrace {
    uint64_t profile_fingerprint = 0;
    int tokens = 0;
    int num_layers = 0;
    int experts_per_layer = 0;
    int top_k = 0;
    std::vector<int32_t> slots;

    const int32_t* record(int token, int layer) const {
        return slots.data() + (static_cast<size_t>(token) * num_layers + layer) * top_k;
    }
    friend bool operator==(const GatingTrace&, const GatingTrace&) = default;
};

GatingTrace generate_trace(const ModelProfile& profile, int tokens, uint64_t seed);
std::string write_trace(const GatingTrace& trace);
GatingTrace read_trace(std::string_view document);

}  // namespace moeb200
