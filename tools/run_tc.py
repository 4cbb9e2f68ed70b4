"""Run a few eager batched (tcgen05) decode steps, for ncu captures.
usage: python tools/run_tc.py [n4] [T] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_14417_b200 as moe  # noqa: E402

n4 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(32, 8, 2, 4096, 14336, plan, max_tokens=T, seed=0, norm_eps=1e-5, tc_min_tokens=32,
                    use_graphs=False)
eng.synth_input(0, T)
for _ in range(steps):
    eng.decode(T)
eng.sync()
eng.close()
print("ok")
