"""Batched-decode (tcgen05 path) step rate per plan: tok/s and the expert
bytes each step streams (distinct selected experts per layer, from the
routing).  usage: python tools/tc_tps.py [n4 list] [T list]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_14417_b200 as moe  # noqa: E402

n4s = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,128,256").split(",")]
Ts = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "64,256").split(",")]
prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
s16, s4 = moe.expert_size(prof, 1), moe.expert_size(prof, 0)
for n4 in n4s:
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(32, 8, 2, 4096, 14336, plan, max_tokens=max(Ts), seed=0, norm_eps=1e-5, tc_min_tokens=32)
    for T in Ts:
        eng.synth_input(0, T)
        eng.decode(T)
        eng.sync()
        ms = bench.time_engine(moe, torch, eng, T, 16, 3)
        r = eng.last_routing(T)
        b = 0
        for l in range(32):
            sel = {r[(t * 32 + l) * 2 + j] for t in range(T) for j in range(2)}
            b += sum(s16 if plan.precision[l * 8 + s] == 1 else s4 for s in sel)
        print(f"n4={n4:3d} T={T:3d}  {T * 1000 / ms:8.1f} tok/s  {ms:7.2f} ms/step  {b / ms / 1e6:7.1f} GB/s "
              f"({b / 1e9:.1f} GB/step)", flush=True)
    eng.close()
