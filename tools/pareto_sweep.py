"""Measured Pareto sweep: the reference's `pareto` subcommand (cli.cpp:293-350,
options cli.cpp:424-434) over the engine's Mixtral shape, with measured decode
tok/s and hit rate appended to every feasible row.

usage: python tools/pareto_sweep.py [--mem-range 24GB:96GB:24GB] [--n4-grid 0,128,256]
         [--tokens 200] [--seed 0] [--dataset wikitext2] [--steps 16] [--no-measure]
         [--bw BYTES_PER_S] [--out FILE]

Without --bw the transfer bandwidth of the simulated columns is the measured
pinned H2D copy rate of this GPU (so both columns price the same link);
with --no-measure only the reference table is produced (no GPU needed).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2407_14417_b200 as moe  # noqa: E402
from paper_2407_14417_b200 import pareto  # noqa: E402

SHAPE = (32, 8, 2, 4096, 14336)  # Mixtral-8x7B: L, E, k, d, f


def h2d_bytes_per_s(nbytes=1 << 30):
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3))
    return best


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--mem-range", default="24GB:96GB:24GB")
    ap.add_argument("--n4-grid", default="0,128,256")
    ap.add_argument("--tokens", type=int, default=200, help="simulated tokens per cell")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dataset", default="wikitext2")
    ap.add_argument("--steps", type=int, default=16, help="measured decode steps per distinct placement")
    ap.add_argument("--bw", type=float, default=None)
    ap.add_argument("--no-measure", action="store_true")
    ap.add_argument("--shape", default=",".join(map(str, SHAPE)))
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    shape = tuple(int(v) for v in a.shape.split(","))
    budgets = pareto.parse_mem_range(moe, a.mem_range)
    grid = pareto.parse_n4_grid(moe, a.n4_grid)
    bw = a.bw if a.bw else (moe.HardwareProfile(1).transfer_bw_bytes_per_s if a.no_measure else h2d_bytes_per_s())
    rows, meas = pareto.measured_sweep(moe, budgets, grid, shape, bw, a.tokens, a.seed, moe.builtin_anchors(a.dataset),
                                       a.steps, measure=not a.no_measure)
    doc = moe.pareto_csv(rows, None if a.no_measure else meas)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(doc)
        print(f"pareto: rows={len(rows)} frontier={sum(r.on_frontier for r in rows)} bw={bw / 1e9:.1f}GB/s")
    else:
        sys.stdout.write(doc)


if __name__ == "__main__":
    main()
