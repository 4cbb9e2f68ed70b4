"""Measured Pareto sweep.

The reference's `pareto` subcommand (cli.cpp:293-350) sweeps GPU-memory
budgets x n4. For each cell it plans with the quality preference, simulates
the Static policy on one generated trace (sweep_memory,
simulator.cpp:139-163), attaches the perplexity surrogate, marks the
frontier, and prints the table of cli.cpp:253-270.

This module builds the same table through the C ABI (pareto_sweep /
pareto_csv, which are bit-identical to the reference). For every feasible cell
it then runs the engine on the GPU with that cell's placement and reports the
measured decode tok/s and the engine's own hit rate next to the simulated
columns:

- device-resident experts run from HBM;
- host-resident experts stream from the pinned arena into the swap slot on
  every activation, exactly as the Static policy models it.

Cells with the same placement share one measurement.
"""
from __future__ import annotations

import re
import time
from typing import List, Optional, Sequence, Tuple


def parse_mem_range(moe, spec: str) -> List[int]:
    """`FROM:TO:STEP` or a single size (cli.cpp:52-72)."""
    parts = spec.split(":")
    if len(parts) == 1:
        return [moe.parse_size(parts[0])]
    if len(parts) != 3:
        raise moe.UsageError(2, f"--mem-range expects FROM:TO:STEP (or a single size), got '{spec}'")
    lo, hi, step = (moe.parse_size(p) for p in parts)
    if step <= 0:
        raise moe.UsageError(2, "--mem-range step must be positive")
    if hi < lo:
        raise moe.UsageError(2, "--mem-range upper bound below lower bound")
    return list(range(lo, hi + 1, step))


def parse_n4_grid(moe, spec: str) -> List[int]:
    """Comma-separated non-negative integers (cli.cpp:74-91)."""
    grid = []
    for item in spec.split(","):
        # std::stoi: leading whitespace and a sign, then digits to the end
        if not re.fullmatch(r"\s*[+-]?\d+", item) or int(item) < 0:
            raise moe.UsageError(2, f"--n4-grid expects comma-separated non-negative integers, got '{item}'")
        grid.append(int(item))
    if not grid:
        raise moe.UsageError(2, "--n4-grid must not be empty")
    return grid


def measure_cell(moe, plan, shape: Tuple[int, int, int, int, int], steps: int, seed: int, device: int = 0,
                 norm_eps: float = 1e-5, lru_capacity: int = 0) -> Tuple[float, float]:
    """Decode `steps` single-token steps with `plan`'s placement.

    Returns (tokens/s, hit rate). The time is wall-clock around the
    synchronised steps, so it includes the host -> device expert streaming.
    The hit rate comes from the engine's counters, which equal simulate() on
    the same routing (tests/test_gpu_engine.py)."""
    L, E, k, d, f = shape
    eng = moe.MoeEngine(L, E, k, d, f, plan, max_tokens=1, seed=seed, device=device, norm_eps=norm_eps,
                        use_graphs=True, lru_capacity=lru_capacity)
    try:
        eng.synth_input(0, 1)
        eng.decode(1)
        eng.sync()
        eng.reset_counters()
        t0 = time.perf_counter()
        for s in range(steps):
            eng.synth_input(s + 1, 1)
            eng.decode(1)
        eng.sync()
        el = time.perf_counter() - t0
        c = eng.counters()
        return steps / el, c.hit_rate
    finally:
        eng.close()


def measured_sweep(moe, budgets: Sequence[int], n4_grid: Sequence[int], shape, hw_bw: float, tokens: int = 200,
                   seed: int = 0, anchors=None, steps: int = 16, device: int = 0,
                   measure: bool = True) -> Tuple[list, List[Optional[Tuple[float, float]]]]:
    """pareto_sweep rows for the engine's shape, plus per-row measurements."""
    L, E, k, d, f = shape
    prof = moe.profile_for_shape(d, f, L, E, k)
    rows = moe.pareto_sweep(budgets, n4_grid, prof, moe.HardwareProfile(1, hw_bw), tokens, seed, anchors)
    measured: List[Optional[Tuple[float, float]]] = [None] * len(rows)
    if not measure:
        return rows, measured
    cache = {}
    for i, r in enumerate(rows):
        if not r.feasible:
            continue
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, r.n4, seed), moe.HardwareProfile(r.budget, hw_bw), prof)
        key = (tuple(plan.precision), tuple(plan.location))
        if key not in cache:
            cache[key] = measure_cell(moe, plan, shape, steps, seed, device)
        measured[i] = cache[key]
    return rows, measured
