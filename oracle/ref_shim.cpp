// ref_shim.cpp -- extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp), compiled in place by oracle/Makefile into
// oracle/_ref/libmoeserve_ref.so.  TEST INFRASTRUCTURE ONLY: it is the checker
// for the product's planner / trace / counter re-implementation and the
// "model" column of bench.py; the product never links it.
//
// Wrapped reference entry points:
//   make_plan            planner.hpp:71   (planner.cpp:137-141)
//   num_experts_16       planner.hpp:52   (planner.cpp:33-41)
//   assign_locations     planner.hpp:61   (planner.cpp:57-110)
//   generate_trace       gating.hpp:33    (gating.cpp:31-53)
//   write/read_trace     gating.hpp:38-43 (gating.cpp:55-188)
//   simulate             simulator.hpp:58 (simulator.cpp:66-112)
//   expected_throughput  simulator.hpp:64 (simulator.cpp:114-137)
//   load_profiles        profiles.hpp:84  (profiles.cpp:148-211)
//   expert_size / model_size / profile_fingerprint (profiles.cpp:221-256)
//   diff_plans / estimate_cost (reconfig.cpp:19-82)
//   write_plan / read_plan (serialize.cpp:99-149, when built with nlohmann)
//   anchors / ppl_estimate / n4_for_budget / frontier_mask (pareto.cpp) and
//   the `pareto` sweep rows (cli.cpp:308-342 restated over sweep_memory,
//   simulator.cpp:139-163 -- cli.cpp itself needs CLI11)
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "moeserve/errors.hpp"
#include "moeserve/gating.hpp"
#include "moeserve/pareto.hpp"
#include "moeserve/planner.hpp"
#include "moeserve/profiles.hpp"
#include "moeserve/reconfig.hpp"
#include "moeserve/simulator.hpp"
#ifdef REF_HAVE_SERIALIZE
#include "moeserve/serialize.hpp"
#endif

using namespace moeserve;

extern "C" {

struct ref_profile {
    int32_t num_layers, experts_per_layer, top_k, pad_;
    int64_t size_nonexpert_bytes, size_expert16_bytes;
    double quant_ratio, compute_latency16_s, compute_penalty4, nonexpert_latency_s;
};

}  // extern "C"

namespace {

thread_local std::string g_err;

ModelProfile to_model(const ref_profile* p) {
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

void from_model(const ModelProfile& m, ref_profile* p) {
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

HardwareProfile to_hw(int64_t gpu_mem, double bw) {
    HardwareProfile hw;
    hw.gpu_mem_bytes = gpu_mem;
    hw.transfer_bw_bytes_per_s = bw;
    return hw;
}

// exit-code convention of cli.hpp:7-8
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const UsageError& e) {
        g_err = e.what();
        return 2;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 3;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return 3;
    } catch (const InfeasibleError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

PlacementPlan to_plan(const int32_t* prec, const int32_t* loc, int n, int64_t swap, uint64_t seed) {
    PlacementPlan plan;
    plan.entries.resize(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        plan.entries[i].precision = prec[i] == 0 ? Precision::P4 : Precision::P16;
        plan.entries[i].location = loc[i] == 0 ? Location::GPU : Location::CPU;
    }
    plan.swap_slot_bytes = swap;
    plan.seed = seed;
    return plan;
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

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_default_profile(int which, ref_profile* out) {
    from_model(which == 1 ? mixtral_table1() : mixtral_sec41(), out);
}

int ref_load_profiles(const char* doc, ref_profile* out, int64_t* gpu_mem, double* bw) {
    return guarded([&] {
        const auto [m, hw] = load_profiles(doc);
        from_model(m, out);
        *gpu_mem = hw.gpu_mem_bytes;
        *bw = hw.transfer_bw_bytes_per_s;
    });
}

int64_t ref_expert_size(const ref_profile* p, int precision) {
    return expert_size(to_model(p), precision == 0 ? Precision::P4 : Precision::P16);
}

int ref_model_size(const ref_profile* p, int n4, int nonexpert_precision, int64_t* out) {
    return guarded([&] {
        const NonexpertPrecision np = nonexpert_precision == 0   ? NonexpertPrecision::P4
                                      : nonexpert_precision == 1 ? NonexpertPrecision::P8
                                                                 : NonexpertPrecision::P16;
        *out = model_size(to_model(p), n4, np);
    });
}

uint64_t ref_profile_fingerprint(const ref_profile* p) { return profile_fingerprint(to_model(p)); }

int ref_num_experts_16(const ref_profile* p, int64_t mem) { return num_experts_16(mem, to_model(p)); }

int ref_make_plan(const ref_profile* p, int64_t gpu_mem, double bw, int preference, int n4_target,
                  uint64_t seed, int32_t* prec_out, int32_t* loc_out, int64_t* swap_out) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        TaskRequest task;
        task.preference = preference == 0 ? Preference::Throughput : Preference::Quality;
        if (n4_target >= -1000 && n4_target != -1) task.n4_target = n4_target;
        task.seed = seed;
        const PlacementPlan plan = make_plan(task, to_hw(gpu_mem, bw), m);
        for (size_t i = 0; i < plan.entries.size(); ++i) {
            prec_out[i] = plan.entries[i].precision == Precision::P4 ? 0 : 1;
            loc_out[i] = plan.entries[i].location == Location::GPU ? 0 : 1;
        }
        *swap_out = plan.swap_slot_bytes;
    });
}

int ref_assign_locations(const ref_profile* p, int64_t gpu_mem, double bw, const int32_t* prec,
                         uint64_t seed, int32_t* loc_out, int64_t* swap_out) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        std::vector<Precision> pv(static_cast<size_t>(m.num_experts()));
        for (size_t i = 0; i < pv.size(); ++i) pv[i] = prec[i] == 0 ? Precision::P4 : Precision::P16;
        const PlacementPlan plan = assign_locations(pv, to_hw(gpu_mem, bw), m, seed);
        for (size_t i = 0; i < plan.entries.size(); ++i)
            loc_out[i] = plan.entries[i].location == Location::GPU ? 0 : 1;
        *swap_out = plan.swap_slot_bytes;
    });
}

int ref_generate_trace(const ref_profile* p, int tokens, uint64_t seed, int32_t* slots_out,
                       uint64_t* fingerprint_out) {
    return guarded([&] {
        const GatingTrace tr = generate_trace(to_model(p), tokens, seed);
        std::memcpy(slots_out, tr.slots.data(), tr.slots.size() * sizeof(int32_t));
        *fingerprint_out = tr.profile_fingerprint;
    });
}

// Writes the v1 text of a trace into buf (capacity cap); returns the length
// (or the required length when cap is too small), -1 on error.
int64_t ref_write_trace(const ref_profile* p, int tokens, const int32_t* slots, char* buf,
                        int64_t cap) {
    std::string s;
    if (guarded([&] { s = write_trace(to_trace(to_model(p), tokens, slots)); }) != 0) return -1;
    if (static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int64_t>(s.size());
}

// Parses a v1 document; returns status, fills dims and (when slots_out is
// non-null and large enough) the slots.
int ref_read_trace(const char* doc, int32_t dims[4], uint64_t* fingerprint, int32_t* slots_out,
                   int64_t slots_cap) {
    return guarded([&] {
        const GatingTrace tr = read_trace(doc);
        dims[0] = tr.tokens;
        dims[1] = tr.num_layers;
        dims[2] = tr.experts_per_layer;
        dims[3] = tr.top_k;
        *fingerprint = tr.profile_fingerprint;
        if (slots_out && static_cast<int64_t>(tr.slots.size()) <= slots_cap)
            std::memcpy(slots_out, tr.slots.data(), tr.slots.size() * sizeof(int32_t));
    });
}

// out = {activations, hits, bytes_transferred, transfer_ns, compute_ns, nonexpert_ns}
int ref_simulate(const ref_profile* p, double bw, const int32_t* prec, const int32_t* loc,
                 int64_t swap, uint64_t plan_seed, int tokens, const int32_t* slots,
                 int lru_capacity, int64_t out[6]) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        const PlacementPlan plan = to_plan(prec, loc, m.num_experts(), swap, plan_seed);
        const ResidencyPolicy pol =
            lru_capacity > 0 ? ResidencyPolicy::lru(lru_capacity) : ResidencyPolicy::static_policy();
        const SimReport r = simulate(plan, to_trace(m, tokens, slots), m, to_hw(1, bw), pol);
        out[0] = r.activations;
        out[1] = r.hits;
        out[2] = r.bytes_transferred;
        out[3] = r.transfer_ns;
        out[4] = r.compute_ns;
        out[5] = r.nonexpert_ns;
    });
}

double ref_expected_throughput(const ref_profile* p, double bw, const int32_t* prec,
                               const int32_t* loc, int64_t swap) {
    double v = -1.0;
    guarded([&] {
        const ModelProfile m = to_model(p);
        v = expected_throughput(to_plan(prec, loc, m.num_experts(), swap, 0), m, to_hw(1, bw));
    });
    return v;
}

// Reconfiguration diff (control plane, §8f row f1): returns the number of
// actions (kinds: 0 Offload, 1 Fetch, 2 Quantize, 3 Dequantize) written into
// kinds/experts (capacity cap), bytes moved and downtime.
int ref_diff_plans(const ref_profile* p, double bw, const int32_t* prec_a, const int32_t* loc_a,
                   const int32_t* prec_b, const int32_t* loc_b, int32_t* kinds, int32_t* experts,
                   int cap, int64_t* bytes, double* downtime) {
    int n = -1;
    const int st = guarded([&] {
        const ModelProfile m = to_model(p);
        const auto a = to_plan(prec_a, loc_a, m.num_experts(), required_swap_bytes(to_plan(prec_a, loc_a, m.num_experts(), 0, 0), m), 0);
        const auto b = to_plan(prec_b, loc_b, m.num_experts(), required_swap_bytes(to_plan(prec_b, loc_b, m.num_experts(), 0, 0), m), 0);
        const ReconfigPlan rp = diff_plans(a, b, m, to_hw(1, bw));
        n = static_cast<int>(rp.actions.size());
        for (int i = 0; i < n && i < cap; ++i) {
            kinds[i] = static_cast<int32_t>(rp.actions[i].kind);
            experts[i] = expert_index(m, rp.actions[i].expert);
        }
        *bytes = rp.bytes_moved;
        *downtime = rp.est_downtime_s;
    });
    return st == 0 ? n : -st;
}

// Full action lists: 5 int32 per action (kind, layer, slot, target precision
// 0 P4 / 1 P16, target location 0 GPU / 1 CPU).
int ref_reconfig_diff(const ref_profile* p, double bw, const int32_t* prec_a, const int32_t* loc_a,
                      const int32_t* prec_b, const int32_t* loc_b, uint64_t seed_b, int32_t* acts, int cap,
                      int64_t* bytes, double* downtime) {
    int n = -1;
    const int st = guarded([&] {
        const ModelProfile m = to_model(p);
        const auto a = to_plan(prec_a, loc_a, m.num_experts(), 0, 0);
        const auto b = to_plan(prec_b, loc_b, m.num_experts(), 0, seed_b);
        const ReconfigPlan rp = diff_plans(a, b, m, to_hw(1, bw));
        n = static_cast<int>(rp.actions.size());
        for (int i = 0; i < n && i < cap; ++i) {
            const ReconfigAction& x = rp.actions[static_cast<size_t>(i)];
            acts[5 * i + 0] = static_cast<int32_t>(x.kind);
            acts[5 * i + 1] = x.expert.layer;
            acts[5 * i + 2] = x.expert.slot;
            acts[5 * i + 3] = x.target_precision == Precision::P4 ? 0 : 1;
            acts[5 * i + 4] = x.target_location == Location::GPU ? 0 : 1;
        }
        *bytes = rp.bytes_moved;
        *downtime = rp.est_downtime_s;
    });
    return st == 0 ? n : -st;
}

int ref_reconfig_apply(const ref_profile* p, const int32_t* prec, const int32_t* loc, uint64_t seed,
                       const int32_t* acts, int n, uint64_t target_seed, int64_t budget, int32_t* out_prec,
                       int32_t* out_loc, int64_t* out_swap, uint64_t* out_seed) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        PlacementPlan plan = to_plan(prec, loc, m.num_experts(), 0, seed);
        plan.swap_slot_bytes = required_swap_bytes(plan, m);
        ReconfigPlan rp;
        rp.target_seed = target_seed;
        for (int i = 0; i < n; ++i) {
            ReconfigAction a;
            a.kind = static_cast<ActionKind>(acts[5 * i]);
            a.expert = ExpertId{acts[5 * i + 1], acts[5 * i + 2]};
            a.target_precision = acts[5 * i + 3] == 0 ? Precision::P4 : Precision::P16;
            a.target_location = acts[5 * i + 4] == 0 ? Location::GPU : Location::CPU;
            rp.actions.push_back(a);
        }
        const HardwareProfile hw = to_hw(budget, 1.0);
        const PlacementPlan r = apply(plan, rp, m, budget > 0 ? &hw : nullptr);
        for (size_t i = 0; i < r.entries.size(); ++i) {
            out_prec[i] = r.entries[i].precision == Precision::P4 ? 0 : 1;
            out_loc[i] = r.entries[i].location == Location::GPU ? 0 : 1;
        }
        *out_swap = r.swap_slot_bytes;
        *out_seed = r.seed;
    });
}

// ---- pareto (same row layout as moe_pareto_row in include/moe_b200.h)
struct ref_pareto_row {
    int64_t budget;
    int32_t n4, feasible, on_frontier, n_gpu;
    int64_t gpu_bytes;
    double ppl;
    int64_t tokens, activations, hits, bytes_transferred, transfer_ns, compute_ns, nonexpert_ns;
};

int ref_builtin_anchors(const char* name, double* p16, double* p4) {
    return guarded([&] {
        const auto a = builtin_anchors(name);
        if (!a) throw UsageError("unknown dataset");
        *p16 = a->ppl_all16;
        *p4 = a->ppl_all4;
    });
}

int ref_load_anchors(const char* doc, double* p16, double* p4) {
    return guarded([&] {
        const QualityAnchors a = load_anchors(doc, QualityAnchors{"", *p16, *p4});
        *p16 = a.ppl_all16;
        *p4 = a.ppl_all4;
    });
}

int ref_ppl_estimate(int n4, double p16, double p4, int num_e, double* out) {
    return guarded([&] { *out = ppl_estimate(n4, QualityAnchors{"", p16, p4}, num_e); });
}

int ref_n4_for_budget(double budget, double p16, double p4, int num_e, int32_t* out) {
    return guarded([&] { *out = n4_for_budget(budget, QualityAnchors{"", p16, p4}, num_e); });
}

int ref_frontier_mask(int n, const double* tps, const double* ppl, const int64_t* gpu_bytes, int32_t* out) {
    return guarded([&] {
        std::vector<ParetoPoint> pts(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) pts[static_cast<size_t>(i)] = {0, 0, tps[i], ppl[i], gpu_bytes[i]};
        const auto m = frontier_mask(pts);
        for (int i = 0; i < n; ++i) out[i] = m[static_cast<size_t>(i)];
    });
}

int ref_pareto_sweep(const ref_profile* p, double bw, const int64_t* budgets, int nb, const int32_t* grid, int ng,
                     int tokens, uint64_t seed, double p16, double p4, ref_pareto_row* rows) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        const QualityAnchors anchors{"", p16, p4};
        const std::vector<bytes_t> bl(budgets, budgets + nb);
        std::vector<ref_pareto_row> out;
        std::vector<SimReport> reps;
        for (int g = 0; g < ng; ++g) {
            TaskRequest task;
            task.preference = Preference::Quality;
            task.n4_target = grid[g];
            task.seed = seed;
            const double ppl = ppl_estimate(grid[g], anchors, m.num_experts());
            for (const SweepEntry& e : sweep_memory(bl, task, m, to_hw(1, bw), tokens, seed)) {
                ref_pareto_row r{};
                r.budget = e.budget;
                r.n4 = grid[g];
                r.feasible = e.feasible;
                r.n_gpu = e.summary.n_gpu;
                r.gpu_bytes = e.summary.gpu_bytes;
                r.ppl = ppl;
                r.tokens = e.report.tokens;
                r.activations = e.report.activations;
                r.hits = e.report.hits;
                r.bytes_transferred = e.report.bytes_transferred;
                r.transfer_ns = e.report.transfer_ns;
                r.compute_ns = e.report.compute_ns;
                r.nonexpert_ns = e.report.nonexpert_ns;
                out.push_back(r);
                reps.push_back(e.report);
            }
        }
        std::vector<ParetoPoint> pts;
        std::vector<size_t> at;
        for (size_t i = 0; i < out.size(); ++i) {
            if (!out[i].feasible) continue;
            pts.push_back({out[i].budget, out[i].n4, reps[i].throughput_tps(), out[i].ppl, out[i].gpu_bytes});
            at.push_back(i);
        }
        const auto mask = frontier_mask(pts);
        for (size_t i = 0; i < pts.size(); ++i) out[at[i]].on_frontier = mask[i];
        std::memcpy(rows, out.data(), out.size() * sizeof(ref_pareto_row));
    });
}

#ifdef REF_HAVE_SERIALIZE
// Plan JSON (serialize.cpp:99-149).  Returns the document length (copied
// when it fits `cap`), or -status on error.
int64_t ref_write_plan(const ref_profile* p, const int32_t* prec, const int32_t* loc, uint64_t seed, int64_t swap,
                       char* buf, int64_t cap) {
    int64_t n = -1;
    const int st = guarded([&] {
        const ModelProfile m = to_model(p);
        PlacementPlan plan = to_plan(prec, loc, m.num_experts(), swap, seed);
        const std::string doc = write_plan(plan, m);
        n = static_cast<int64_t>(doc.size());
        if (buf != nullptr && n < cap) std::memcpy(buf, doc.c_str(), doc.size() + 1);
    });
    return st == 0 ? n : -st;
}

int ref_read_plan(const char* doc, const ref_profile* p, int32_t* prec, int32_t* loc, uint64_t* seed,
                  int64_t* swap) {
    return guarded([&] {
        const ModelProfile m = to_model(p);
        const PlacementPlan plan = read_plan(doc, m);
        for (size_t i = 0; i < plan.entries.size(); ++i) {
            prec[i] = static_cast<int32_t>(plan.entries[i].precision);
            loc[i] = static_cast<int32_t>(plan.entries[i].location);
        }
        *seed = plan.seed;
        *swap = plan.swap_slot_bytes;
    });
}

// write_reconfig(diff_plans(a, b)) and read_reconfig; 5 int32 per action as
// ref_reconfig_diff.
int64_t ref_write_reconfig(const ref_profile* p, double bw, const int32_t* prec_a, const int32_t* loc_a,
                           const int32_t* prec_b, const int32_t* loc_b, uint64_t seed_b, char* buf, int64_t cap) {
    int64_t n = -1;
    const int st = guarded([&] {
        const ModelProfile m = to_model(p);
        const ReconfigPlan rp = diff_plans(to_plan(prec_a, loc_a, m.num_experts(), 0, 0),
                                           to_plan(prec_b, loc_b, m.num_experts(), 0, seed_b), m, to_hw(1, bw));
        const std::string doc = write_reconfig(rp, m);
        n = static_cast<int64_t>(doc.size());
        if (buf != nullptr && n < cap) std::memcpy(buf, doc.c_str(), doc.size() + 1);
    });
    return st == 0 ? n : -st;
}

int ref_read_reconfig(const char* doc, const ref_profile* p, double bw, int32_t* acts, int cap, int* n,
                      uint64_t* seed, int64_t* bytes, double* downtime) {
    return guarded([&] {
        const ReconfigPlan rp = read_reconfig(doc, to_model(p), to_hw(1, bw));
        *n = static_cast<int>(rp.actions.size());
        for (int i = 0; i < *n && i < cap; ++i) {
            const ReconfigAction& x = rp.actions[static_cast<size_t>(i)];
            acts[5 * i + 0] = static_cast<int32_t>(x.kind);
            acts[5 * i + 1] = x.expert.layer;
            acts[5 * i + 2] = x.expert.slot;
            acts[5 * i + 3] = x.target_precision == Precision::P4 ? 0 : 1;
            acts[5 * i + 4] = x.target_location == Location::GPU ? 0 : 1;
        }
        *seed = rp.target_seed;
        *bytes = rp.bytes_moved;
        *downtime = rp.est_downtime_s;
    });
}

// report_csv / report_json of a SimReport given by its counters.
int64_t ref_report_text(const int64_t* c, int json, char* buf, int64_t cap) {
    int64_t n = -1;
    const int st = guarded([&] {
        SimReport r;
        r.tokens = static_cast<int>(c[0]);
        r.activations = c[1];
        r.hits = c[2];
        r.bytes_transferred = c[3];
        r.transfer_ns = c[4];
        r.compute_ns = c[5];
        r.nonexpert_ns = c[6];
        const std::string doc = json ? report_json(r) : report_csv(r);
        n = static_cast<int64_t>(doc.size());
        if (buf != nullptr && n < cap) std::memcpy(buf, doc.c_str(), doc.size() + 1);
    });
    return st == 0 ? n : -st;
}

int ref_have_serialize(void) { return 1; }
#else
int ref_have_serialize(void) { return 0; }
#endif

}  // extern "C"
