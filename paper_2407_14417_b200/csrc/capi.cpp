// capi.cu -- the extern "C" boundary (include/moe_b200.h).
//
// Status codes mirror the reference CLI's exit codes (cli.hpp:7-8,
// cli.cpp:473-488): exceptions of the reference's four error types map to
// 2 (usage), 3 (parse/validation), 4 (infeasible); CUDA and other failures
// to 1.  No entry point falls back to the CPU.
#include <cuda_runtime.h>

#include <cstring>
#include <exception>
#include <string>

#include "kernels/launch.h"
#include "moe_b200.h"
#include "moeb200/engine.hpp"
#include "moeb200/reconfig.hpp"
#include "moeb200/serialize.hpp"
#include "moeb200/pareto.hpp"

using namespace moeb200;

namespace moeb200 {
int weight_shift(int K);
}

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return MOE_OK;
    } catch (const UsageError& e) {
        g_err = e.what();
        return MOE_ERR_USAGE;
    } catch (const ParseError& e) {
        g_err = e.what();
        return MOE_ERR_VALIDATION;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return MOE_ERR_VALIDATION;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return MOE_ERR_INFEASIBLE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MOE_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return MOE_ERR_INTERNAL;
    }
}

void usage_if(bool bad, const std::string& msg) {
    if (bad) throw UsageError(msg);
}

ModelProfile to_model(const moe_model_profile* p) {
    usage_if(p == nullptr, "null model profile");
    ModelProfile m;
    m.num_layers = p->num_layers;
    m.experts_per_layer = p->experts_per_layer;
    m.top_k = p->top_k;
    m.size_nonexpert_bytes = p->size_nonexpert_bytes;
    m.size_expert16_bytes = p->size_expert16_bytes;
    m.quant_ratio = p->quant_ratio;
    m.compute_latency16_s = p->compute_latency16_s;
    m.compute_penalty4 = p->compute_penalty4;
    m.nonexpert_latency_s = p->nonexpert_latency_s;
    return m;
}

void from_model(const ModelProfile& m, moe_model_profile* p) {
    std::memset(p, 0, sizeof *p);
    p->num_layers = m.num_layers;
    p->experts_per_layer = m.experts_per_layer;
    p->top_k = m.top_k;
    p->size_nonexpert_bytes = m.size_nonexpert_bytes;
    p->size_expert16_bytes = m.size_expert16_bytes;
    p->quant_ratio = m.quant_ratio;
    p->compute_latency16_s = m.compute_latency16_s;
    p->compute_penalty4 = m.compute_penalty4;
    p->nonexpert_latency_s = m.nonexpert_latency_s;
}

HardwareProfile to_hw(const moe_hardware_profile* h) {
    usage_if(h == nullptr, "null hardware profile");
    HardwareProfile hw;
    hw.gpu_mem_bytes = h->gpu_mem_bytes;
    hw.transfer_bw_bytes_per_s = h->transfer_bw_bytes_per_s;
    return hw;
}

PlacementPlan to_plan(const moe_expert_state* entries, int n, int64_t swap) {
    PlacementPlan plan;
    plan.entries.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        plan.entries[static_cast<size_t>(i)].precision = entries[i].precision == MOE_P4 ? Precision::P4 : Precision::P16;
        plan.entries[static_cast<size_t>(i)].location = entries[i].location == MOE_GPU ? Location::GPU : Location::CPU;
    }
    plan.swap_slot_bytes = swap;
    return plan;
}

void from_plan(const PlacementPlan& plan, moe_expert_state* entries, int64_t* swap) {
    for (size_t i = 0; i < plan.entries.size(); ++i) {
        entries[i].precision = plan.entries[i].precision == Precision::P4 ? MOE_P4 : MOE_P16;
        entries[i].location = plan.entries[i].location == Location::GPU ? MOE_GPU : MOE_CPU;
    }
    if (swap) *swap = plan.swap_slot_bytes;
}

GatingTrace to_trace(const ModelProfile& m, int tokens, const int32_t* slots) {
    GatingTrace tr;
    tr.profile_fingerprint = profile_fingerprint(m);
    tr.tokens = tokens;
    tr.num_layers = m.num_layers;
    tr.experts_per_layer = m.experts_per_layer;
    tr.top_k = m.top_k;
    tr.slots.assign(slots, slots + static_cast<size_t>(tokens) * m.num_layers * m.top_k);
    return tr;
}

void need_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw std::runtime_error("no CUDA device: kernels have no CPU fallback");
    const cudaError_t e = moek_numerics_bind_device();
    if (e != cudaSuccess) throw std::runtime_error(std::string("numerics guard: ") + cudaGetErrorString(e));
}

cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

struct moe_engine {
    MoeEngine* impl;
};

extern "C" {

const char* moe_last_error(void) { return g_err.c_str(); }
int moe_version(void) { return 1; }

int moe_profile_builtin(int which, moe_model_profile* out) {
    return guarded([&] {
        usage_if(which != 0 && which != 1, "builtin profile must be 0 (mixtral-sec41) or 1 (mixtral-table1)");
        from_model(which == 0 ? mixtral_sec41() : mixtral_table1(), out);
    });
}

int moe_profile_for_shape(int d_model, int d_ffn, int num_layers, int experts_per_layer, int top_k,
                          int64_t size_nonexpert_bytes, moe_model_profile* out) {
    return guarded([&] {
        MoeShape s;
        s.d_model = d_model;
        s.d_ffn = d_ffn;
        const ModelProfile m = profile_for_shape(s, num_layers, experts_per_layer, top_k, size_nonexpert_bytes);
        validate_profile(m);
        from_model(m, out);
    });
}

int moe_load_profiles(const char* document, moe_model_profile* model, moe_hardware_profile* hw) {
    return guarded([&] {
        usage_if(document == nullptr, "null document");
        const auto [m, h] = load_profiles(document);
        from_model(m, model);
        hw->gpu_mem_bytes = h.gpu_mem_bytes;
        hw->transfer_bw_bytes_per_s = h.transfer_bw_bytes_per_s;
    });
}

int64_t moe_parse_size(const char* text) {
    int64_t v = -1;
    if (guarded([&] { v = parse_size(text ? text : ""); }) != MOE_OK) return -1;
    return v;
}

int64_t moe_expert_size(const moe_model_profile* p, int precision) {
    int64_t v = -1;
    guarded([&] { v = expert_size(to_model(p), precision == MOE_P4 ? Precision::P4 : Precision::P16); });
    return v;
}

int moe_model_size(const moe_model_profile* p, int n4, int nonexpert_precision, int64_t* out) {
    return guarded([&] {
        const NonexpertPrecision np = nonexpert_precision == 0   ? NonexpertPrecision::P4
                                      : nonexpert_precision == 1 ? NonexpertPrecision::P8
                                                                 : NonexpertPrecision::P16;
        *out = model_size(to_model(p), n4, np);
    });
}

uint64_t moe_profile_fingerprint(const moe_model_profile* p) {
    uint64_t v = 0;
    guarded([&] { v = profile_fingerprint(to_model(p)); });
    return v;
}

int moe_num_experts_16(int64_t mem_gpu, const moe_model_profile* p) {
    int v = -1;
    guarded([&] { v = num_experts_16(mem_gpu, to_model(p)); });
    return v;
}

int moe_make_plan(const moe_task_request* task, const moe_hardware_profile* hw,
                  const moe_model_profile* p, moe_expert_state* entries, int64_t* swap_slot_bytes) {
    return guarded([&] {
        usage_if(task == nullptr || entries == nullptr, "null argument");
        TaskRequest t;
        t.preference = task->preference == MOE_QUALITY ? Preference::Quality : Preference::Throughput;
        if (task->n4_target != -1) t.n4_target = task->n4_target;
        t.seed = task->seed;
        from_plan(make_plan(t, to_hw(hw), to_model(p)), entries, swap_slot_bytes);
    });
}

int moe_assign_locations(const int32_t* precisions, const moe_hardware_profile* hw,
                         const moe_model_profile* p, uint64_t seed, moe_expert_state* entries,
                         int64_t* swap_slot_bytes) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        std::vector<Precision> prec(static_cast<size_t>(m.num_experts()));
        for (size_t i = 0; i < prec.size(); ++i) prec[i] = precisions[i] == MOE_P4 ? Precision::P4 : Precision::P16;
        from_plan(assign_locations(prec, to_hw(hw), m, seed), entries, swap_slot_bytes);
    });
}

int64_t moe_gpu_footprint(const moe_expert_state* entries, int64_t swap_slot_bytes,
                          const moe_model_profile* p) {
    int64_t v = -1;
    guarded([&] {
        const ModelProfile m = to_model(p);
        v = gpu_footprint(to_plan(entries, m.num_experts(), swap_slot_bytes), m);
    });
    return v;
}

int moe_validate_plan(const moe_expert_state* entries, int n_entries, int64_t swap_slot_bytes,
                      const moe_hardware_profile* hw, const moe_model_profile* p, char* msg, int cap) {
    int n = -1;
    guarded([&] {
        const auto v = validate_plan(to_plan(entries, n_entries, swap_slot_bytes), to_hw(hw), to_model(p));
        n = static_cast<int>(v.size());
        if (msg && cap > 0) {
            std::string all;
            for (const auto& s : v) all += s + "\n";
            std::strncpy(msg, all.c_str(), static_cast<size_t>(cap - 1));
            msg[cap - 1] = 0;
        }
    });
    return n;
}

int moe_generate_trace(const moe_model_profile* p, int tokens, uint64_t seed, int32_t* slots,
                       uint64_t* fingerprint) {
    return guarded([&] {
        const GatingTrace tr = generate_trace(to_model(p), tokens, seed);
        std::memcpy(slots, tr.slots.data(), tr.slots.size() * 4);
        if (fingerprint) *fingerprint = tr.profile_fingerprint;
    });
}

int64_t moe_write_plan(const moe_expert_state* entries, int64_t swap_slot_bytes, uint64_t seed,
                       const moe_model_profile* p, char* buf, int64_t cap) {
    std::string s;
    if (guarded([&] {
            usage_if(entries == nullptr, "null argument");
            const ModelProfile m = to_model(p);
            PlacementPlan plan = to_plan(entries, m.num_experts(), swap_slot_bytes);
            plan.seed = seed;
            s = write_plan(plan, m);
        }) != MOE_OK)
        return -1;
    if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

int moe_read_plan(const char* document, const moe_model_profile* p, moe_expert_state* entries,
                  int64_t* swap_slot_bytes, uint64_t* seed) {
    return guarded([&] {
        usage_if(entries == nullptr, "null argument");
        const PlacementPlan plan = read_plan(document ? document : "", to_model(p));
        from_plan(plan, entries, swap_slot_bytes);
        if (seed) *seed = plan.seed;
    });
}

int64_t moe_write_trace(const moe_model_profile* p, int tokens, const int32_t* slots, char* buf,
                        int64_t cap) {
    std::string s;
    if (guarded([&] { s = write_trace(to_trace(to_model(p), tokens, slots)); }) != MOE_OK) return -1;
    if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

int moe_read_trace(const char* document, int32_t dims[4], uint64_t* fingerprint, int32_t* slots,
                   int64_t slots_cap) {
    return guarded([&] {
        const GatingTrace tr = read_trace(document ? document : "");
        dims[0] = tr.tokens;
        dims[1] = tr.num_layers;
        dims[2] = tr.experts_per_layer;
        dims[3] = tr.top_k;
        if (fingerprint) *fingerprint = tr.profile_fingerprint;
        if (slots && static_cast<int64_t>(tr.slots.size()) <= slots_cap)
            std::memcpy(slots, tr.slots.data(), tr.slots.size() * 4);
    });
}

int moe_simulate(const moe_expert_state* entries, int64_t swap_slot_bytes, const int32_t* slots,
                 int tokens, const moe_model_profile* p, const moe_hardware_profile* hw,
                 int lru_capacity, moe_sim_report* out) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        const ResidencyPolicy pol = lru_capacity > 0 ? ResidencyPolicy::lru(lru_capacity) : ResidencyPolicy::static_policy();
        const SimReport r = simulate(to_plan(entries, m.num_experts(), swap_slot_bytes), to_trace(m, tokens, slots),
                                     m, to_hw(hw), pol);
        out->tokens = r.tokens;
        out->activations = r.activations;
        out->hits = r.hits;
        out->bytes_transferred = r.bytes_transferred;
        out->transfer_ns = r.transfer_ns;
        out->compute_ns = r.compute_ns;
        out->nonexpert_ns = r.nonexpert_ns;
    });
}

double moe_expected_throughput(const moe_expert_state* entries, const moe_model_profile* p,
                               const moe_hardware_profile* hw) {
    double v = -1.0;
    guarded([&] {
        const ModelProfile m = to_model(p);
        v = expected_throughput(to_plan(entries, m.num_experts(), 0), m, to_hw(hw));
    });
    return v;
}

namespace {

ReconfigPlan to_reconfig(const moe_reconfig_action* acts, int n, uint64_t target_seed) {
    ReconfigPlan rp;
    rp.target_seed = target_seed;
    for (int i = 0; i < n; ++i) {
        const moe_reconfig_action& c = acts[i];
        usage_if(c.kind < 0 || c.kind > 3, "unknown action kind");
        ReconfigAction a;
        a.kind = static_cast<ActionKind>(c.kind);
        a.expert = ExpertId{c.layer, c.slot};
        a.target_precision = c.target_precision == MOE_P4 ? Precision::P4 : Precision::P16;
        a.target_location = c.target_location == MOE_GPU ? Location::GPU : Location::CPU;
        rp.actions.push_back(a);
    }
    return rp;
}

}  // namespace

namespace {

int64_t copy_text(const std::string& s, char* buf, int64_t cap) {
    if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

}  // namespace

int64_t moe_write_reconfig(const moe_reconfig_action* actions, int n_actions, uint64_t target_seed,
                           const moe_model_profile* p, const moe_hardware_profile* hw, char* buf, int64_t cap) {
    std::string s;
    if (guarded([&] {
            usage_if(n_actions > 0 && actions == nullptr, "null argument");
            const ModelProfile m = to_model(p);
            ReconfigPlan rp = to_reconfig(actions, n_actions, target_seed);
            std::tie(rp.bytes_moved, rp.est_downtime_s) = estimate_cost(rp, m, to_hw(hw));
            s = write_reconfig(rp, m);
        }) != MOE_OK)
        return -1;
    return copy_text(s, buf, cap);
}

int moe_read_reconfig(const char* document, const moe_model_profile* p, const moe_hardware_profile* hw,
                      moe_reconfig_action* actions, int cap, int* n_actions, uint64_t* target_seed,
                      int64_t* bytes_moved, double* est_downtime_s) {
    return guarded([&] {
        usage_if(n_actions == nullptr, "null argument");
        const ReconfigPlan rp = read_reconfig(document ? document : "", to_model(p), to_hw(hw));
        *n_actions = static_cast<int>(rp.actions.size());
        for (int i = 0; i < *n_actions && i < cap && actions; ++i) {
            const ReconfigAction& x = rp.actions[static_cast<size_t>(i)];
            actions[i] = {static_cast<int32_t>(x.kind), x.expert.layer, x.expert.slot,
                          x.target_precision == Precision::P4 ? MOE_P4 : MOE_P16,
                          x.target_location == Location::GPU ? MOE_GPU : MOE_CPU, 0};
        }
        if (target_seed) *target_seed = rp.target_seed;
        if (bytes_moved) *bytes_moved = rp.bytes_moved;
        if (est_downtime_s) *est_downtime_s = rp.est_downtime_s;
    });
}

int64_t moe_report_text(const moe_sim_report* r, int json, char* buf, int64_t cap) {
    std::string s;
    if (guarded([&] {
            usage_if(r == nullptr, "null argument");
            SimReport x;
            x.tokens = static_cast<int>(r->tokens);
            x.activations = r->activations;
            x.hits = r->hits;
            x.bytes_transferred = r->bytes_transferred;
            x.transfer_ns = r->transfer_ns;
            x.compute_ns = r->compute_ns;
            x.nonexpert_ns = r->nonexpert_ns;
            s = json ? report_json(x) : report_csv(x);
        }) != MOE_OK)
        return -1;
    return copy_text(s, buf, cap);
}

int moe_diff_plans(const moe_expert_state* from, const moe_expert_state* to, uint64_t to_seed,
                   const moe_model_profile* p, const moe_hardware_profile* hw, moe_reconfig_action* actions,
                   int cap, int* n_actions, int64_t* bytes_moved, double* est_downtime_s) {
    return guarded([&] {
        usage_if(from == nullptr || to == nullptr || n_actions == nullptr, "null argument");
        const ModelProfile m = to_model(p);
        const PlacementPlan a = to_plan(from, m.num_experts(), 0);
        PlacementPlan b = to_plan(to, m.num_experts(), 0);
        b.seed = to_seed;
        const ReconfigPlan rp = diff_plans(a, b, m, to_hw(hw));
        *n_actions = static_cast<int>(rp.actions.size());
        for (int i = 0; i < *n_actions && i < cap && actions; ++i) {
            const ReconfigAction& x = rp.actions[static_cast<size_t>(i)];
            actions[i] = {static_cast<int32_t>(x.kind), x.expert.layer, x.expert.slot,
                          x.target_precision == Precision::P4 ? MOE_P4 : MOE_P16,
                          x.target_location == Location::GPU ? MOE_GPU : MOE_CPU, 0};
        }
        if (bytes_moved) *bytes_moved = rp.bytes_moved;
        if (est_downtime_s) *est_downtime_s = rp.est_downtime_s;
    });
}

int moe_apply_reconfig(const moe_expert_state* plan, uint64_t plan_seed, const moe_reconfig_action* actions,
                       int n_actions, uint64_t target_seed, const moe_model_profile* p,
                       const moe_hardware_profile* budget, moe_expert_state* out, int64_t* out_swap,
                       uint64_t* out_seed) {
    return guarded([&] {
        usage_if(plan == nullptr || out == nullptr || (n_actions > 0 && actions == nullptr), "null argument");
        const ModelProfile m = to_model(p);
        PlacementPlan pl = to_plan(plan, m.num_experts(), 0);
        pl.swap_slot_bytes = required_swap_bytes(pl, m);
        pl.seed = plan_seed;
        const HardwareProfile hb = budget ? to_hw(budget) : HardwareProfile{};
        const PlacementPlan r = apply(pl, to_reconfig(actions, n_actions, target_seed), m, budget ? &hb : nullptr);
        from_plan(r, out, out_swap);
        if (out_seed) *out_seed = r.seed;
    });
}

namespace {

QualityAnchors anchors_of(double p16, double p4) { return QualityAnchors{"", p16, p4}; }

void to_c_report(const SimReport& r, moe_sim_report* out) {
    *out = {r.tokens, r.activations, r.hits, r.bytes_transferred, r.transfer_ns, r.compute_ns, r.nonexpert_ns};
}

ParetoRow from_c_row(const moe_pareto_row& c) {
    ParetoRow r;
    r.budget = c.budget;
    r.n4 = c.n4;
    r.feasible = c.feasible != 0;
    r.on_frontier = c.on_frontier != 0;
    r.summary.n_gpu = c.n_gpu;
    r.summary.gpu_bytes = c.gpu_bytes;
    r.ppl = c.ppl;
    const moe_sim_report& s = c.report;
    r.report.tokens = static_cast<int>(s.tokens);
    r.report.activations = s.activations;
    r.report.hits = s.hits;
    r.report.bytes_transferred = s.bytes_transferred;
    r.report.transfer_ns = s.transfer_ns;
    r.report.compute_ns = s.compute_ns;
    r.report.nonexpert_ns = s.nonexpert_ns;
    return r;
}

}  // namespace

int moe_builtin_anchors(const char* name, double* ppl_all16, double* ppl_all4) {
    return guarded([&] {
        const auto a = builtin_anchors(name ? name : "");
        usage_if(!a, std::string("unknown dataset '") + (name ? name : "") + "' (known: wikitext2, ptb, c4)");
        *ppl_all16 = a->ppl_all16;
        *ppl_all4 = a->ppl_all4;
    });
}

int moe_load_anchors(const char* document, double* ppl_all16, double* ppl_all4) {
    return guarded([&] {
        const QualityAnchors a = load_anchors(document ? document : "", anchors_of(*ppl_all16, *ppl_all4));
        *ppl_all16 = a.ppl_all16;
        *ppl_all4 = a.ppl_all4;
    });
}

int moe_ppl_estimate(int n4, double ppl_all16, double ppl_all4, int num_e, double* out) {
    return guarded([&] { *out = ppl_estimate(n4, anchors_of(ppl_all16, ppl_all4), num_e); });
}

int moe_n4_for_budget(double ppl_budget, double ppl_all16, double ppl_all4, int num_e, int32_t* out) {
    return guarded([&] { *out = n4_for_budget(ppl_budget, anchors_of(ppl_all16, ppl_all4), num_e); });
}

int moe_pareto_sweep(const int64_t* budgets, int n_budgets, const int32_t* n4_grid, int n_grid,
                     const moe_model_profile* p, const moe_hardware_profile* hw, int tokens, uint64_t seed,
                     double ppl_all16, double ppl_all4, moe_pareto_row* rows) {
    return guarded([&] {
        usage_if(rows == nullptr || n_budgets < 0 || n_grid < 0, "bad sweep arguments");
        const std::vector<bytes_t> b(budgets, budgets + n_budgets);
        const std::vector<int> g(n4_grid, n4_grid + n_grid);
        const auto out = pareto_sweep(b, g, to_model(p), to_hw(hw), tokens, seed, anchors_of(ppl_all16, ppl_all4));
        for (size_t i = 0; i < out.size(); ++i) {
            const ParetoRow& r = out[i];
            moe_pareto_row& c = rows[i];
            c = {};
            c.budget = r.budget;
            c.n4 = r.n4;
            c.feasible = r.feasible;
            c.on_frontier = r.on_frontier;
            c.n_gpu = r.summary.n_gpu;
            c.gpu_bytes = r.summary.gpu_bytes;
            c.ppl = r.ppl;
            to_c_report(r.report, &c.report);
        }
    });
}

int moe_frontier_mask(int n, const double* throughput_tps, const double* ppl, const int64_t* gpu_bytes,
                      int32_t* on_frontier) {
    return guarded([&] {
        std::vector<ParetoPoint> pts(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) pts[static_cast<size_t>(i)] = {0, 0, throughput_tps[i], ppl[i], gpu_bytes[i]};
        const auto m = frontier_mask(pts);
        for (int i = 0; i < n; ++i) on_frontier[i] = m[static_cast<size_t>(i)];
    });
}

int64_t moe_pareto_csv(const moe_pareto_row* rows, int n, const double* measured, char* buf, int64_t cap) {
    std::string s;
    if (guarded([&] {
            std::vector<ParetoRow> r;
            std::vector<MeasuredCell> m;
            for (int i = 0; i < n; ++i) {
                r.push_back(from_c_row(rows[i]));
                if (measured) m.push_back({measured[2 * i], measured[2 * i + 1]});
            }
            s = pareto_csv(r, measured ? &m : nullptr);
        }) != MOE_OK)
        return -1;
    if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

// ---------------------------------------------------------------- kernels
int moe_gate_topk(const void* x, const void* wg, int T, int d, int E, int k, int32_t* idx,
                  float* w, float* logits, void* stream) {
    return guarded([&] {
        usage_if(T < 0 || d <= 0 || d % 8 != 0, "d must be a positive multiple of 8");
        usage_if(E < 1 || E > MOE_MAX_EXPERTS || k < 1 || k > E || k > MOE_MAX_TOPK, "bad E / k");
        need_device();
        if (T == 0) return;
        const cudaError_t e = moek_route(x, wg, T, d, E, k, idx, w, logits, nullptr, nullptr, nullptr,
                                         nullptr, nullptr, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_gate_topk: ") + cudaGetErrorString(e));
    });
}

int moe_route(const void* x, const void* wg, int T, int d, int E, int k, float norm_eps, int32_t* idx, float* w,
              float* logits, int32_t* counts, int32_t* offsets, int32_t* perm, int32_t* inv_perm, void* xnat,
              uint32_t* ticket, void* stream) {
    return guarded([&] {
        usage_if(T < 0 || d <= 0 || d % 8 != 0, "d must be a positive multiple of 8");
        usage_if(E < 1 || E > MOE_MAX_EXPERTS || k < 1 || k > E || k > MOE_MAX_TOPK, "bad E / k");
        usage_if(!(norm_eps >= 0.0f), "norm_eps must be >= 0");
        usage_if(counts != nullptr && (offsets == nullptr || perm == nullptr || inv_perm == nullptr || ticket == nullptr),
                 "the fused permutation needs offsets, perm, inv_perm and a zeroed ticket");
        need_device();
        if (T == 0) return;
        const cudaError_t e = moek_route(x, wg, T, d, E, k, idx, w, logits, counts, offsets, perm, inv_perm, ticket,
                                         st(stream), nullptr, nullptr, nullptr, 0, norm_eps, xnat);
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_route: ") + cudaGetErrorString(e));
    });
}

int moe_combine_partial(const float* y_perm, const int32_t* inv_perm, const float* w, const int32_t* idx,
                        uint64_t expert_mask, int T, int d, int k, float* out, void* stream) {
    return guarded([&] {
        usage_if(T < 0 || d <= 0 || d % 4 != 0 || k < 1, "bad T / d / k");
        need_device();
        const cudaError_t e = moek_combine_partial(y_perm, inv_perm, w, idx, expert_mask, T, d, k, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_combine_partial: ") + cudaGetErrorString(e));
    });
}

int moe_residual_add(const void* residual, const float* part, int64_t n, void* out, void* stream) {
    return guarded([&] {
        usage_if(n < 0, "bad n");
        need_device();
        const cudaError_t e = moek_residual_add(residual, part, n, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_residual_add: ") + cudaGetErrorString(e));
    });
}

int moe_permute(const int32_t* idx, int T, int E, int k, int32_t* counts, int32_t* offsets,
                int32_t* perm, int32_t* inv_perm, void* stream) {
    return guarded([&] {
        usage_if(T < 0 || E < 1 || E > MOE_MAX_EXPERTS || k < 1 || k > E, "bad T / E / k");
        need_device();
        const cudaError_t e = moek_permute(idx, T, E, k, counts, offsets, perm, inv_perm, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_permute: ") + cudaGetErrorString(e));
    });
}

int moe_numerics_status(int clear, uint32_t* flags) {
    return guarded([&] {
        usage_if(flags == nullptr, "flags is null");
        *flags = moek_numerics_status(clear);
    });
}

int moe_gemv_max_tokens(int E, int k) { return moek_gemv_max_tokens(E, k); }

size_t moe_ffn_workspace_bytes(int T, int k, int E, int d, int f) {
    if (T < 1 || k < 1 || E < 1 || d < 128 || f < 128) return 0;
    return moek_gemv_workspace_bytes(T, k, d, f);
}

int moe_ffn(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
            const moe_expert_weights* experts, int E, int d, int f, void* workspace, size_t ws_bytes,
            float* y_perm, void* stream) {
    return guarded([&] {
        usage_if(E < 1 || E > MOE_MAX_EXPERTS || k < 1 || k > E, "bad E / k");
        usage_if(d <= 0 || d % 256 != 0 || f <= 0 || f % 128 != 0,
                 "d must be a multiple of 256 and f a multiple of 128");
        need_device();
        if (T == 0) return;
        usage_if(T > moek_gemv_max_tokens(E, k), "T exceeds moe_gemv_max_tokens(E, k): use moe_ffn_tc");
        usage_if(workspace == nullptr || ws_bytes < moek_gemv_workspace_bytes(T, k, d, f),
                 "workspace too small (moe_ffn_workspace_bytes)");
        const GemvWorkspace ws = moek_gemv_workspace_view(workspace, T, k, d, f);
        uint64_t mask = 0;  // experts without weights (another rank's shard) are skipped
        for (int i = 0; i < E; ++i)
            if (experts[i].w_gate_up != nullptr) mask |= 1ull << i;
        const cudaError_t e = moek_ffn_mma(ws, x, perm, offsets, nullptr, nullptr, nullptr, T, k, experts, E, d, f,
                                           mask, nullptr, y_perm, MOE_X_PERMUTE, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_ffn: ") + cudaGetErrorString(e));
    });
}

size_t moe_ffn_tc_workspace_bytes(int T, int k, int d, int f) { return moek_tc_workspace_bytes(T, k, d, f); }

int moe_ffn_tc(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
               const moe_expert_weights* experts, int E, int d, int f, void* workspace, size_t ws_bytes,
               float* y_perm, void* stream) {
    return guarded([&] {
        usage_if(E < 1 || E > MOE_MAX_EXPERTS || k < 1 || k > E, "bad E / k");
        usage_if(d <= 0 || d % 128 != 0 || f <= 0 || f % 128 != 0, "d and f must be multiples of 128");
        need_device();
        if (T == 0) return;
        usage_if(workspace == nullptr || ws_bytes < moek_tc_workspace_bytes(T, k, d, f),
                 "workspace too small (moe_ffn_tc_workspace_bytes)");
        uint64_t mask = 0;  // experts without weights (another rank's shard) are skipped
        for (int i = 0; i < E; ++i)
            if (experts[i].w_gate_up != nullptr) mask |= 1ull << i;
        const cudaError_t e = moek_ffn_tc(workspace, x, perm, offsets, T, k, experts, E, d, f, mask, y_perm, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_ffn_tc: ") + cudaGetErrorString(e));
    });
}

int moe_ffn_int4(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                 const void* const* q_gate_up, const void* const* s_gate_up,
                 const void* const* q_down, const void* const* s_down, int E, int d, int f,
                 void* workspace, size_t ws_bytes, float* y_perm, void* stream) {
    moe_expert_weights ex[MOE_MAX_EXPERTS];
    if (E < 1 || E > MOE_MAX_EXPERTS) {
        g_err = "bad E";
        return MOE_ERR_USAGE;
    }
    for (int e = 0; e < E; ++e) ex[e] = {MOE_P4, 0, q_gate_up[e], s_gate_up[e], q_down[e], s_down[e]};
    return moe_ffn(x, perm, offsets, T, k, ex, E, d, f, workspace, ws_bytes, y_perm, stream);
}

int moe_ffn_bf16(const void* x, const int32_t* perm, const int32_t* offsets, int T, int k,
                 const void* const* w_gate_up, const void* const* w_down, int E, int d, int f,
                 void* workspace, size_t ws_bytes, float* y_perm, void* stream) {
    moe_expert_weights ex[MOE_MAX_EXPERTS];
    if (E < 1 || E > MOE_MAX_EXPERTS) {
        g_err = "bad E";
        return MOE_ERR_USAGE;
    }
    for (int e = 0; e < E; ++e) ex[e] = {MOE_P16, 0, w_gate_up[e], nullptr, w_down[e], nullptr};
    return moe_ffn(x, perm, offsets, T, k, ex, E, d, f, workspace, ws_bytes, y_perm, stream);
}

int moe_combine(const float* y_perm, const int32_t* inv_perm, const float* w, const void* residual,
                int T, int d, int k, void* out, void* stream) {
    return guarded([&] {
        usage_if(T < 0 || d <= 0 || d % 4 != 0 || k < 1, "bad T / d / k");
        need_device();
        const cudaError_t e = moek_combine(y_perm, inv_perm, w, residual, T, d, k, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_combine: ") + cudaGetErrorString(e));
    });
}

int moe_quantize_g128(const void* w, int rows, int cols, uint32_t* q, void* s, void* stream) {
    return guarded([&] {
        usage_if(rows < 0 || rows % 16 != 0 || cols <= 0 || cols % 128 != 0,
                 "rows must be a multiple of 16 and cols a positive multiple of 128");
        need_device();
        const cudaError_t e = moek_quantize_blocks(w, rows, cols, q, s, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_quantize_g128: ") + cudaGetErrorString(e));
    });
}

int moe_pack_bf16_blocks(const void* w, int rows, int cols, void* out, void* stream) {
    return guarded([&] {
        usage_if(rows < 0 || rows % 16 != 0 || cols <= 0 || cols % 128 != 0,
                 "rows must be a multiple of 16 and cols a positive multiple of 128");
        need_device();
        const cudaError_t e = moek_pack_bf16_blocks(w, rows, cols, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_pack_bf16_blocks: ") + cudaGetErrorString(e));
    });
}

int moe_synth_weight_bf16(uint64_t seed, uint64_t uid, int64_t n, int shift, void* out, void* stream) {
    return guarded([&] {
        need_device();
        const cudaError_t e = moek_synth_weight(seed, uid, n, shift, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    });
}

int moe_synth_input_bf16(uint64_t seed, uint64_t uid, int64_t n, void* out, void* stream) {
    return guarded([&] {
        need_device();
        const cudaError_t e = moek_synth_input(seed, uid, n, out, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    });
}

int moe_weight_shift(int K) { return weight_shift(K); }

int moe_stream_expert(void* dst_dev, const void* src_pinned, size_t bytes, void* copy_stream,
                      void* done_event) {
    return guarded([&] {
        usage_if(bytes > 0 && (dst_dev == nullptr || src_pinned == nullptr), "null buffer");
        need_device();
        const cudaError_t e = moek_stream_expert(dst_dev, src_pinned, bytes, st(copy_stream),
                                                 static_cast<cudaEvent_t>(done_event));
        if (e != cudaSuccess) throw std::runtime_error(std::string("moe_stream_expert: ") + cudaGetErrorString(e));
    });
}

// ---------------------------------------------------------------- engine
int moe_engine_create(const moe_engine_config* cfg, const moe_expert_state* plan_entries,
                      moe_engine** out) {
    return guarded([&] {
        usage_if(cfg == nullptr || plan_entries == nullptr || out == nullptr, "null argument");
        MoeShape shape;
        shape.d_model = cfg->d_model;
        shape.d_ffn = cfg->d_ffn;
        EngineConfig ec;
        ec.shape = shape;
        ec.profile = profile_for_shape(shape, cfg->num_layers, cfg->experts_per_layer, cfg->top_k, 1);
        ec.max_tokens = cfg->max_tokens;
        ec.seed = cfg->seed;
        ec.device = cfg->device;
        ec.use_graphs = cfg->use_graphs != 0;
        ec.per_layer_decode = cfg->per_layer_decode != 0;
        usage_if(!(cfg->norm_eps >= 0.0f), "norm_eps must be >= 0");
        ec.norm_eps = cfg->norm_eps;
        usage_if(cfg->tc_min_tokens < 0, "tc_min_tokens must be >= 0");
        ec.tc_min_tokens = cfg->tc_min_tokens > 0 ? cfg->tc_min_tokens : 32;
        usage_if(cfg->lru_capacity < 0, "lru_capacity must be >= 0");
        ec.lru_capacity = cfg->lru_capacity;
        ec.keep_masters = cfg->keep_masters != 0;
        ec.ep_rank = cfg->ep_world > 1 ? cfg->ep_rank : 0;
        ec.ep_world = cfg->ep_world > 1 ? cfg->ep_world : 1;
        const int n = cfg->num_layers * cfg->experts_per_layer;
        PlacementPlan plan = to_plan(plan_entries, n, 0);
        plan.swap_slot_bytes = required_swap_bytes(plan, ec.profile);
        *out = new moe_engine{new MoeEngine(ec, plan)};
    });
}

int moe_engine_ep_buffer(moe_engine* eng, void** base, int64_t* bytes) {
    return guarded([&] {
        usage_if(eng == nullptr || base == nullptr, "null argument");
        size_t b = 0;
        *base = eng->impl->ep_buffer(&b);
        if (bytes) *bytes = static_cast<int64_t>(b);
    });
}

int moe_engine_ep_set_peers(moe_engine* eng, const void* const* bases, int32_t world) {
    return guarded([&] {
        usage_if(eng == nullptr, "null argument");
        eng->impl->ep_set_peers(bases, world);
    });
}

void moe_engine_destroy(moe_engine* eng) {
    if (!eng) return;
    delete eng->impl;
    delete eng;
}

int moe_engine_memory(const moe_engine* eng, int64_t* expert_bytes, int64_t* swap_bytes,
                      int64_t* host_pinned_bytes, int64_t* workspace_bytes) {
    return guarded([&] { eng->impl->memory(expert_bytes, swap_bytes, host_pinned_bytes, workspace_bytes); });
}

void* moe_engine_input(moe_engine* eng) { return eng ? eng->impl->input() : nullptr; }
void* moe_engine_output(moe_engine* eng) { return eng ? eng->impl->output() : nullptr; }
void* moe_engine_stream(moe_engine* eng) { return eng ? eng->impl->stream() : nullptr; }

int moe_engine_synth_input(moe_engine* eng, int step, int T) {
    return guarded([&] { eng->impl->synth_input(step, T); });
}

int moe_engine_decode(moe_engine* eng, int T) {
    return guarded([&] { eng->impl->decode(T); });
}

int moe_engine_decode_host(moe_engine* eng, const void* x_host, int T, void* out_host) {
    return guarded([&] { eng->impl->decode_host(x_host, T, out_host); });
}

int moe_engine_forward_layer(moe_engine* eng, int layer, const void* x, int T, void* out,
                             int32_t* idx_dev, float* w_dev, float* logits_dev) {
    return guarded([&] { eng->impl->forward_layer(layer, x, T, out, idx_dev, w_dev, logits_dev); });
}

int moe_engine_sync(moe_engine* eng) {
    return guarded([&] { eng->impl->sync(); });
}

int moe_engine_profile_step(moe_engine* eng, int T, float* ffn_ms, int64_t* ffn_bytes,
                            int32_t* kernels_per_step) {
    return guarded([&] {
        int k = 0;
        eng->impl->profile_step(T, ffn_ms, ffn_bytes, &k);
        if (kernels_per_step) *kernels_per_step = k;
    });
}

int moe_debug_engine_buffer(moe_engine* eng, int which, void** ptr, size_t* bytes) {
    return guarded([&] { *ptr = eng->impl->debug_buffer(which, bytes); });
}

int moe_debug_fused_trace(void* buf) {
    return guarded([&] {
        need_device();
        const cudaError_t e = moek_debug_fused_trace(buf);
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    });
}

int moe_engine_profile_fused(moe_engine* eng, float* ms, int64_t* bytes) {
    return guarded([&] {
        usage_if(ms == nullptr || bytes == nullptr, "null output");
        usage_if(!eng->impl->profile_fused(ms, bytes), "the engine does not use the fused batch-1 step");
    });
}

int moe_engine_last_routing(moe_engine* eng, int T, int32_t* slots_out) {
    return guarded([&] {
        const GatingTrace tr = eng->impl->last_routing(T);
        std::memcpy(slots_out, tr.slots.data(), tr.slots.size() * 4);
    });
}

int moe_engine_reconfigure(moe_engine* eng, const moe_expert_state* target, uint64_t target_seed,
                           double transfer_bw_bytes_per_s, moe_reconfig_report* out) {
    return guarded([&] {
        usage_if(eng == nullptr || target == nullptr, "null argument");
        usage_if(!(transfer_bw_bytes_per_s > 0.0), "transfer bandwidth must be > 0");
        const PlacementPlan& cur = eng->impl->plan();
        PlacementPlan t = to_plan(target, static_cast<int>(cur.entries.size()), 0);
        t.seed = target_seed;
        HardwareProfile hw;
        hw.transfer_bw_bytes_per_s = transfer_bw_bytes_per_s;
        const ReconfigReport r = eng->impl->reconfigure(t, hw);
        if (out) *out = {r.actions, 0, r.bytes_moved, r.est_downtime_s, r.bytes_h2d, r.measured_s};
    });
}

namespace {
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace

size_t moe_ep_peer_bytes(int G, int T_local, int d) { return moek_ep_peer_bytes(G, T_local, d); }

void* moe_ep_peer_rows(void* base) { return base; }  // the gather rows lead the buffer

int moe_ep_peer_alloc(size_t bytes, void** base) {
    return guarded([&] {
        usage_if(base == nullptr || bytes == 0, "bad argument");
        need_device();
        cuda_ok(cudaMalloc(base, bytes), "cudaMalloc(exchange buffer)");
        cuda_ok(cudaMemset(*base, 0, bytes), "cudaMemset");
    });
}

int moe_ep_peer_free(void* base) {
    return guarded([&] { cuda_ok(cudaFree(base), "cudaFree"); });
}

int moe_ep_peer_ipc_handle(const void* base, char handle[64]) {
    return guarded([&] {
        usage_if(base == nullptr || handle == nullptr, "null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t h;
        cuda_ok(cudaIpcGetMemHandle(&h, const_cast<void*>(base)), "cudaIpcGetMemHandle");
        std::memcpy(handle, &h, sizeof h);
    });
}

int moe_ep_peer_ipc_open(const char handle[64], void** peer_base) {
    return guarded([&] {
        usage_if(handle == nullptr || peer_base == nullptr, "null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof h);
        cuda_ok(cudaIpcOpenMemHandle(peer_base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int moe_ep_peer_ipc_close(void* peer_base) {
    return guarded([&] { cuda_ok(cudaIpcCloseMemHandle(peer_base), "cudaIpcCloseMemHandle"); });
}

int moe_ep_push_rows(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases,
                     uint32_t epoch, void* stream) {
    return guarded([&] {
        usage_if(x_local == nullptr || bases == nullptr || rank < 0 || rank >= G, "bad argument");
        need_device();
        cuda_ok(moek_ep_push_rows(x_local, T_local, d, rank, G, bases, epoch, static_cast<cudaStream_t>(stream)),
                "ep push rows");
    });
}

int moe_ep_wait_rows(const void* my_base, int G, int T_local, int d, uint32_t epoch, void* stream) {
    return guarded([&] {
        usage_if(my_base == nullptr, "null argument");
        need_device();
        cuda_ok(moek_ep_wait_rows(my_base, G, T_local, d, epoch, static_cast<cudaStream_t>(stream)), "ep wait");
    });
}

int moe_ep_push_shares(const float* y_perm, const int32_t* inv_perm, const float* w, const int32_t* idx,
                       uint64_t expert_mask, int T_local, int d, int k, int rank, int G, const void* const* bases,
                       uint32_t epoch, void* stream) {
    return guarded([&] {
        usage_if(y_perm == nullptr || bases == nullptr || rank < 0 || rank >= G, "bad argument");
        need_device();
        cuda_ok(moek_ep_push_shares(y_perm, inv_perm, w, idx, expert_mask, T_local, d, k, rank, G, bases, epoch,
                                    static_cast<cudaStream_t>(stream)),
                "ep push shares");
    });
}

int moe_ep_reduce(const void* x_local, int T_local, int d, int rank, int G, const void* const* bases, uint32_t epoch,
                  void* out, void* stream) {
    return guarded([&] {
        usage_if(x_local == nullptr || out == nullptr || bases == nullptr || rank < 0 || rank >= G, "bad argument");
        need_device();
        cuda_ok(moek_ep_reduce(x_local, T_local, d, rank, G, bases, epoch, out, static_cast<cudaStream_t>(stream)),
                "ep reduce");
    });
}

int moe_engine_counters(const moe_engine* eng, moe_sim_report* out) {
    return guarded([&] {
        const SimReport& r = eng->impl->counters();
        out->tokens = r.tokens;
        out->activations = r.activations;
        out->hits = r.hits;
        out->bytes_transferred = r.bytes_transferred;
        out->transfer_ns = r.transfer_ns;
        out->compute_ns = r.compute_ns;
        out->nonexpert_ns = r.nonexpert_ns;
    });
}

int moe_engine_reset_counters(moe_engine* eng) {
    return guarded([&] { eng->impl->reset_counters(); });
}

int moe_engine_expert(const moe_engine* eng, int layer, int slot, moe_expert_weights* out,
                      int32_t* location) {
    return guarded([&] {
        int loc = 0;
        *out = eng->impl->expert(layer, slot, &loc);
        if (location) *location = loc;
    });
}

int moe_debug_gemv_trace(void* buf) {
    return guarded([&] {
        need_device();
        const cudaError_t e = moek_debug_gemv_trace(buf);
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    });
}

int moe_debug_layer_trace(void* buf, void* stream) {
    return guarded([&] {
        need_device();
        const cudaError_t e = moek_debug_layer_trace(buf, st(stream));
        if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
    });
}

int moe_engine_router(const moe_engine* eng, int layer, const void** wg_dev) {
    return guarded([&] { *wg_dev = eng->impl->router(layer); });
}

}  // extern "C"
