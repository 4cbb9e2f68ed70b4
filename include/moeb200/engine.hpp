// engine.hpp -- MoeEngine: the B200 MoE-layer forward.
//
// Replaces the reference's MoE-layer stand-in simulate() (simulator.hpp:58,
// body simulator.cpp:89-110) with real kernels, keeping its contract:
//   - the expert table comes from a PlacementPlan (planner.hpp:31-36):
//     GPU-resident experts live in HBM at their precision, CPU-resident
//     experts live in a pinned host arena and are streamed into the swap slot
//     (Static policy, simulator.hpp:12-16: every CPU-resident activation is a
//     miss that re-streams the expert) with cudaMemcpyAsync on a side stream;
//     they are never computed on the CPU;
//   - the router is real (K1 top-k softmax) and its decisions are exportable
//     as a GatingTrace (gating.hpp:16-29);
//   - cumulative counters follow SimReport (simulator.hpp:33-53): for the
//     same plan and routing, activations / hits / bytes_transferred equal
//     simulate()'s.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "moe_b200.h"
#include "moeb200/gating.hpp"
#include "moeb200/planner.hpp"
#include "moeb200/reconfig.hpp"
#include "moeb200/simulator.hpp"

namespace moeb200 {

struct EngineConfig {
    ModelProfile profile;     // layers, experts/layer, top_k, byte sizes
    MoeShape shape;           // d_model, d_ffn, group
    int max_tokens = 1;
    uint64_t seed = 0;
    int device = 0;
    bool use_graphs = true;
    float norm_eps = 0.0f;    // > 0: pre-MoE RMSNorm (unit weight), residual = un-normalised x
    int tc_min_tokens = 32;   // T >= this: tcgen05 expert GEMM instead of the streaming GEMV (measured crossover)
    int lru_capacity = 0;     // 0: Static swap slot (simulator.hpp ResidencyPolicy::Static); >0: LRU of that many slots
    bool per_layer_decode = false;  // true: batch-1 decode as 5 launches per layer instead of the fused
                                    // one-launch step (decode_step_kernel); for A/B and the host-split path
    bool keep_masters = false;  // pinned host copy of every expert in both precisions (the reconfig
                                // model's "16-bit master on the CPU", reconfig.hpp:39): required by reconfigure()
    // Expert parallelism: ep_world > 1 shards every layer's
    // experts over ep_world engines (one per GPU, or several on one GPU for
    // tests); this one holds only the slots s with s*ep_world/E == ep_rank.
    // Tokens stay on their rank; each layer sends only the routed rows to the
    // experts' owners and gets their outputs back, over peer memory
    // (ep_set_peers), all inside decode() (graph-captured).
    int ep_rank = 0;
    int ep_world = 1;
};

// What MoeEngine::reconfigure did: the model's numbers (diff_plans) and the
// measured ones.
struct ReconfigReport {
    int actions = 0;
    bytes_t bytes_moved = 0;      // model: CPU -> GPU bytes (estimate_cost)
    double est_downtime_s = 0.0;  // model: bytes_moved / transfer bandwidth
    bytes_t bytes_h2d = 0;        // measured: bytes copied host -> device
    double measured_s = 0.0;      // measured: wall time of the executed action list (synchronised)
};

class MoeEngine {
  public:
    MoeEngine(const EngineConfig& cfg, const PlacementPlan& plan);
    ~MoeEngine();
    MoeEngine(const MoeEngine&) = delete;
    MoeEngine& operator=(const MoeEngine&) = delete;

    void* input();
    void* output();
    void* stream();
    void synth_input(int step, int T);
    // One decode step of T tokens through all layers (async on stream()).
    void decode(int T);
    void decode_host(const void* x_host, int T, void* out_host);
    void forward_layer(int layer, const void* x, int T, void* out, int32_t* idx, float* w,
                       float* logits);
    void sync();
    // Eager step with CUDA events around every layer's expert FFN (see
    // engine.cpp); ffn_ms / ffn_bytes have num_layers entries.
    void profile_step(int T, float* ffn_ms, int64_t* ffn_bytes, int* kernels_per_step);
    // The fused batch-1 step (decode_step_kernel) timed alone: one launch on
    // stream() between CUDA events -> its duration, and the algorithmic bytes
    // it must move (all layers, from the routing it made).  False when the
    // engine does not use the fused step.
    bool profile_fused(float* ms, int64_t* bytes);
    bool fused() const;
    // Debug: device pointer + size of a GEMV workspace buffer (0 part0, 1
    // part1, 2 hperm, 3 hperm16, 4 hsum) for intermediate comparisons.
    void* debug_buffer(int which, size_t* bytes);

    // Executes diff_plans(current plan, target) on the device (SURVEY.md §8f
    // f1): Offload releases the device copy (the expert streams from its host
    // copy afterwards), Fetch copies the host copy at the target precision
    // into HBM, Quantize of a device-resident expert runs the int4-g128
    // quantiser on the device, Dequantize of one pulls its 16-bit master.
    // The replay is checked as apply() does; decode after it is bit-identical
    // to an engine built with `target`.  Needs keep_masters.
    ReconfigReport reconfigure(const PlacementPlan& target, const HardwareProfile& hw);
    const PlacementPlan& plan() const;

    // Expert parallelism: this rank's exchange buffer (its own cudaMalloc
    // allocation, so a CUDA IPC handle maps exactly it) and the G ranks'
    // buffer bases in rank order (this one's included), set before decode.
    void* ep_buffer(size_t* bytes);
    void ep_set_peers(const void* const* bases, int world);

    GatingTrace last_routing(int T);
    const SimReport& counters() const;
    void reset_counters();
    moe_expert_weights expert(int layer, int slot, int* location) const;
    const void* router(int layer) const;
    void memory(int64_t* expert_bytes, int64_t* swap_bytes, int64_t* host_bytes,
                int64_t* workspace_bytes) const;

    struct Impl;

  private:
    std::unique_ptr<Impl> impl_;
};

}  // namespace moeb200
