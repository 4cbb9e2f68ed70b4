// pareto.hpp -- the quality / memory / throughput sweep.
//
// Mirrors the reference's pareto.hpp (quality anchors, the linear perplexity
// surrogate, the dominance frontier) and the table the `pareto` subcommand
// prints (cli.cpp:243-270).  The engine adds one thing the reference cannot
// have: a measured tok/s column next to the simulated one
// (paper_2407_14417_b200/pareto.py drives the GPU cells).
#pragma once

#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "moeb200/config.hpp"
#include "moeb200/planner.hpp"
#include "moeb200/simulator.hpp"

namespace moeb200 {

// Perplexity of one dataset with every expert 16-bit / every expert 4-bit
// (pareto.hpp:14-19; values pareto.cpp:24-26, Table 2).
struct QualityAnchors {
    std::string dataset;
    double ppl_all16 = 0.0;
    double ppl_all4 = 0.0;
};

std::optional<QualityAnchors> builtin_anchors(std::string_view name);  // wikitext2 | ptb | c4
QualityAnchors load_anchors(std::string_view document, const QualityAnchors& fallback);

// Linear interpolation between the anchors at n4 / num_e (pareto.cpp:64-73).
double ppl_estimate(int n4, const QualityAnchors& anchors, int num_e);
// Largest n4 whose estimate is within `ppl_budget` (pareto.cpp:75-93).
int n4_for_budget(double ppl_budget, const QualityAnchors& anchors, int num_e);

struct ParetoPoint {
    bytes_t budget = 0;
    int n4 = 0;
    double throughput_tps = 0.0;
    double ppl_estimate = 0.0;
    bytes_t gpu_bytes = 0;
};
// >= throughput, <= perplexity, <= GPU bytes, strictly better in one.
bool dominates(const ParetoPoint& a, const ParetoPoint& b);
std::vector<char> frontier_mask(const std::vector<ParetoPoint>& points);

// One (budget, n4) cell of the sweep (cli.cpp:243-251).
struct ParetoRow {
    bytes_t budget = 0;
    int n4 = 0;
    bool feasible = false;
    PlanSummary summary;
    SimReport report;
    double ppl = 0.0;
    bool on_frontier = false;
};

// Quality-preference plans over grid x budgets, Static simulate on one
// generated trace, frontier flags over the feasible rows (cli.cpp:308-342).
std::vector<ParetoRow> pareto_sweep(const std::vector<bytes_t>& budgets, const std::vector<int>& n4_grid,
                                    const ModelProfile& profile, const HardwareProfile& hw, int tokens,
                                    uint64_t seed, const QualityAnchors& anchors);

// The reference table (cli.cpp:253-270).  With `measured` (one entry per row,
// NaN = not measured) two columns follow: measured_tps, measured_hit_rate.
struct MeasuredCell {
    double tps = 0.0;
    double hit_rate = 0.0;
};
std::string pareto_csv(const std::vector<ParetoRow>& rows, const std::vector<MeasuredCell>* measured = nullptr);

std::string format_double(double value);  // "%.10g" (serialize.cpp:93-97)

}  // namespace moeb200
