// b200_backend.cpp -- see b200_backend.hpp.
#include "b200_backend.hpp"

#include <stdexcept>
#include <string>

#include "moe_b200.h"
#include "moeserve/errors.hpp"

namespace moeserve::b200 {

void check(int st) {
    if (st == MOE_OK) return;
    const std::string m = moe_last_error();
    switch (st) {
        case MOE_ERR_USAGE: throw UsageError(m);
        case MOE_ERR_VALIDATION: throw ValidationError(m);
        case MOE_ERR_INFEASIBLE: throw InfeasibleError(m);
        default: throw std::runtime_error(m);
    }
}

ModelProfile profile_for_shape(const EngineShape& shape, int num_layers, int experts_per_layer, int top_k,
                               bytes_t size_nonexpert_bytes) {
    moe_model_profile p{};
    check(moe_profile_for_shape(shape.d_model, shape.d_ffn, num_layers, experts_per_layer, top_k,
                                size_nonexpert_bytes, &p));
    ModelProfile m;
    m.num_layers = p.num_layers;
    m.experts_per_layer = p.experts_per_layer;
    m.top_k = p.top_k;
    m.size_nonexpert_bytes = p.size_nonexpert_bytes;
    m.size_expert16_bytes = p.size_expert16_bytes;
    m.quant_ratio = p.quant_ratio;
    m.compute_latency16_s = p.compute_latency16_s;
    m.compute_penalty4 = p.compute_penalty4;
    m.nonexpert_latency_s = p.nonexpert_latency_s;
    return m;
}

SimReport run_engine(const PlacementPlan& plan, const ModelProfile& model, const EngineShape& shape,
                     const ResidencyPolicy& policy, int steps, int T, uint64_t weight_seed,
                     GatingTrace* routing) {
    std::vector<moe_expert_state> st(plan.entries.size());
    for (size_t i = 0; i < st.size(); ++i) {
        st[i].precision = plan.entries[i].precision == Precision::P4 ? MOE_P4 : MOE_P16;
        st[i].location = plan.entries[i].location == Location::GPU ? MOE_GPU : MOE_CPU;
    }
    moe_engine_config cfg{};
    cfg.num_layers = model.num_layers;
    cfg.experts_per_layer = model.experts_per_layer;
    cfg.top_k = model.top_k;
    cfg.d_model = shape.d_model;
    cfg.d_ffn = shape.d_ffn;
    cfg.max_tokens = T;
    cfg.seed = weight_seed;
    cfg.device = 0;
    cfg.use_graphs = 1;
    cfg.norm_eps = shape.norm_eps;
    cfg.lru_capacity = policy.kind == ResidencyPolicy::Kind::Lru ? policy.capacity_slots : 0;
    moe_engine* eng = nullptr;
    check(moe_engine_create(&cfg, st.data(), &eng));
    try {
        std::vector<int32_t> slots(static_cast<size_t>(T) * model.num_layers * model.top_k);
        if (routing) {
            routing->tokens = 0;
            routing->num_layers = model.num_layers;
            routing->experts_per_layer = model.experts_per_layer;
            routing->top_k = model.top_k;
            routing->profile_fingerprint = profile_fingerprint(model);
            routing->slots.clear();
        }
        for (int step = 0; step < steps; ++step) {
            check(moe_engine_synth_input(eng, step, T));  // or copy real embeddings into moe_engine_input()
            check(moe_engine_decode(eng, T));
            if (routing) {
                check(moe_engine_last_routing(eng, T, slots.data()));  // gating.hpp:22 layout
                routing->slots.insert(routing->slots.end(), slots.begin(), slots.end());
                routing->tokens += T;
            }
        }
        check(moe_engine_sync(eng));
        moe_sim_report r{};
        check(moe_engine_counters(eng, &r));
        moe_engine_destroy(eng);
        SimReport out{};
        out.tokens = static_cast<int>(r.tokens);
        out.activations = r.activations;
        out.hits = r.hits;
        out.bytes_transferred = r.bytes_transferred;
        return out;
    } catch (...) {
        moe_engine_destroy(eng);
        throw;
    }
}

}  // namespace moeserve::b200
