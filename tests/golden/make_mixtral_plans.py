"""Freeze the reference planner's plan_quality(n4, seed 0) precisions for the
Mixtral-shaped bench stack (32 x 8 experts) -> tests/golden/mixtral_plans.json.

Run in the container that has /root/reference (oracle/_ref built); bench.py's
--impl reference arm falls back to this file where oracle/_ref is absent.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib, RefProfile  # noqa: E402

L, E, K, D, F = 32, 8, 2, 4096, 14336


def main():
    ref = RefLib()
    prof = RefProfile(L, E, K, 0, 1, 6 * D * F, 128.0 / 33.0, 1e-3, 1.0, 0.0)
    plans = {}
    for n4 in range(0, L * E + 1, 16):
        st, prec, _, _ = ref.make_plan(prof, 10**15, 12.285e9, 1, n4, 0)  # 1 = Quality
        assert st == 0, ref.err()
        plans[str(n4)] = [int(v) for v in prec]
    with open(os.path.join(HERE, "mixtral_plans.json"), "w") as fh:
        json.dump({"source": "oracle/_ref make_plan (planner.cpp:137-141), preference quality, seed 0, "
                             "budget 1e15 (all device-resident)", "plans": plans}, fh)
        fh.write("\n")


if __name__ == "__main__":
    main()
