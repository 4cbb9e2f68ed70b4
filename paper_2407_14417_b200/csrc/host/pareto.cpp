// pareto.cpp -- quality anchors, frontier and the sweep table (see pareto.hpp).
// Behaviour follows the reference (pareto.cpp:24-136, cli.cpp:243-342);
// implementation is independent.
#include "moeb200/pareto.hpp"

#include <cmath>
#include <cstdio>

namespace moeb200 {

namespace {

void check_anchors(const QualityAnchors& a) {
    if (!(a.ppl_all16 > 1.0) || !(a.ppl_all4 > 1.0)) throw ValidationError("perplexity anchors must be > 1");
    if (a.ppl_all4 < a.ppl_all16)
        throw ValidationError(
            "ppl_all4 must be >= ppl_all16 (the surrogate assumes quantization does not improve perplexity)");
}

}  // namespace

std::optional<QualityAnchors> builtin_anchors(std::string_view name) {
    // PAPER.md Table 2 endpoints (all-16-bit / all-4-bit experts)
    struct Row {
        const char* name;
        double p16, p4;
    };
    static constexpr Row kRows[] = {{"wikitext2", 3.81, 4.00}, {"ptb", 13.59, 14.17}, {"c4", 7.24, 7.40}};
    for (const Row& r : kRows)
        if (name == r.name) return QualityAnchors{r.name, r.p16, r.p4};
    return std::nullopt;
}

double ppl_estimate(int n4, const QualityAnchors& anchors, int num_e) {
    check_anchors(anchors);
    if (num_e < 1) throw ValidationError("num_e must be >= 1");
    if (n4 < 0 || n4 > num_e)
        throw ValidationError("n4 out of range: " + std::to_string(n4) + " (expert count " + std::to_string(num_e) +
                              ")");
    const double t = static_cast<double>(n4) / static_cast<double>(num_e);
    return (1.0 - t) * anchors.ppl_all16 + t * anchors.ppl_all4;
}

int n4_for_budget(double ppl_budget, const QualityAnchors& anchors, int num_e) {
    check_anchors(anchors);
    if (num_e < 1) throw ValidationError("num_e must be >= 1");
    if (ppl_budget < anchors.ppl_all16)
        throw ValidationError("perplexity budget " + std::to_string(ppl_budget) + " is below the all-16-bit anchor " +
                              std::to_string(anchors.ppl_all16) + " (unreachable quality)");
    // the estimate is non-decreasing in n4: largest n4 with estimate <= budget
    int lo = 0, hi = num_e;
    while (lo < hi) {
        const int mid = (lo + hi + 1) / 2;
        if (ppl_estimate(mid, anchors, num_e) <= ppl_budget) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

bool dominates(const ParetoPoint& a, const ParetoPoint& b) {
    const bool no_worse = a.throughput_tps >= b.throughput_tps && a.ppl_estimate <= b.ppl_estimate &&
                          a.gpu_bytes <= b.gpu_bytes;
    const bool better = a.throughput_tps > b.throughput_tps || a.ppl_estimate < b.ppl_estimate ||
                        a.gpu_bytes < b.gpu_bytes;
    return no_worse && better;
}

// The definition directly: a point is on the frontier iff nothing dominates
// it.  Sweeps are a few thousand cells at most, so O(n^2) is immaterial.
std::vector<char> frontier_mask(const std::vector<ParetoPoint>& points) {
    std::vector<char> mask(points.size(), 1);
    for (size_t i = 0; i < points.size(); ++i)
        for (size_t j = 0; j < points.size() && mask[i]; ++j)
            if (j != i && dominates(points[j], points[i])) mask[i] = 0;
    return mask;
}

std::vector<ParetoRow> pareto_sweep(const std::vector<bytes_t>& budgets, const std::vector<int>& n4_grid,
                                    const ModelProfile& profile, const HardwareProfile& hw, int tokens,
                                    uint64_t seed, const QualityAnchors& anchors) {
    if (tokens < 1) throw UsageError("--tokens must be >= 1");
    if (n4_grid.empty()) throw UsageError("--n4-grid must not be empty");
    std::vector<ParetoRow> rows;
    for (const int n4 : n4_grid) {
        TaskRequest task;
        task.preference = Preference::Quality;
        task.n4_target = n4;
        task.seed = seed;
        const double ppl = ppl_estimate(n4, anchors, profile.num_experts());
        for (const SweepEntry& e : sweep_memory(budgets, task, profile, hw, tokens, seed)) {
            ParetoRow r;
            r.budget = e.budget;
            r.n4 = n4;
            r.feasible = e.feasible;
            r.summary = e.summary;
            r.report = e.report;
            r.ppl = ppl;
            rows.push_back(r);
        }
    }
    std::vector<ParetoPoint> pts;
    std::vector<size_t> where;
    for (size_t i = 0; i < rows.size(); ++i) {
        if (!rows[i].feasible) continue;
        pts.push_back({rows[i].budget, rows[i].n4, rows[i].report.throughput_tps(), rows[i].ppl,
                       rows[i].summary.gpu_bytes});
        where.push_back(i);
    }
    const std::vector<char> mask = frontier_mask(pts);
    for (size_t i = 0; i < pts.size(); ++i) rows[where[i]].on_frontier = mask[i] != 0;
    return rows;
}

std::string format_double(double value) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.10g", value);
    return buf;
}

std::string pareto_csv(const std::vector<ParetoRow>& rows, const std::vector<MeasuredCell>* measured) {
    std::string out =
        "budget_bytes,n4,n_gpu,gpu_bytes,throughput_tps,hit_rate,bytes_transferred,ppl_estimate,on_frontier,status";
    out += measured ? ",measured_tps,measured_hit_rate\n" : "\n";
    for (size_t i = 0; i < rows.size(); ++i) {
        const ParetoRow& r = rows[i];
        out += std::to_string(r.budget) + ',' + std::to_string(r.n4) + ',';
        if (r.feasible) {
            out += std::to_string(r.summary.n_gpu) + ',' + std::to_string(r.summary.gpu_bytes) + ',' +
                   format_double(r.report.throughput_tps()) + ',' + format_double(r.report.hit_rate()) + ',' +
                   std::to_string(r.report.bytes_transferred) + ',' + format_double(r.ppl) + ',' +
                   (r.on_frontier ? "1" : "0") + ",ok";
        } else {
            out += "-,-,-,-,-," + format_double(r.ppl) + ",0,infeasible";
        }
        if (measured) {
            const MeasuredCell& m = (*measured)[i];
            if (r.feasible && !std::isnan(m.tps))
                out += ',' + format_double(m.tps) + ',' + format_double(m.hit_rate);
            else
                out += ",-,-";
        }
        out += '\n';
    }
    return out;
}

}  // namespace moeb200
