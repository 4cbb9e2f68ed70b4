// b200_backend.hpp -- the binding a moeserve maintainer adds to run
// simulate()'s hot loop on the B200 engine.  Built
// against the reference's own headers (/root/reference/proj/include) and
// linked to libmoe_b200.so; compiled and exercised by
// tests/cpp/boundary_test.cpp (oracle/Makefile `boundary`).
#pragma once

#include <cstdint>
#include <vector>

#include "moeserve/gating.hpp"
#include "moeserve/planner.hpp"
#include "moeserve/simulator.hpp"

namespace moeserve::b200 {

struct EngineShape {
    int d_model = 4096;
    int d_ffn = 14336;
    float norm_eps = 1e-5f;  // Mixtral decoder-layer RMSNorm before each MoE block
};

// Rethrows a C-ABI status as the reference's exceptions (errors.hpp:9-26).
void check(int status);

// ModelProfile whose expert sizes equal the engine's allocations for a
// shape (moe_profile_for_shape): size_expert16 = 6df, quant_ratio = 128/33.
ModelProfile profile_for_shape(const EngineShape& shape, int num_layers, int experts_per_layer, int top_k,
                               bytes_t size_nonexpert_bytes);

// Decode `steps` steps of batch T through the real MoE layers placed by
// `plan` (simulator.hpp:58's contract): the engine's SimReport counters
// (tokens, activations, hits, bytes_transferred) of the real run, and the
// routing it made as a GatingTrace (gating.hpp:16-29) in `routing`.
// policy: Static, or Lru(capacity) -> the engine's LRU device cache.
SimReport run_engine(const PlacementPlan& plan, const ModelProfile& model, const EngineShape& shape,
                     const ResidencyPolicy& policy, int steps, int T, uint64_t weight_seed,
                     GatingTrace* routing);

}  // namespace moeserve::b200
