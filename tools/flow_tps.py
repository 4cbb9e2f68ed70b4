"""tok/s of the fused batch-1 step alone (whatever MOE_FUSED / MOE_BAR_MODE
select), Mixtral shape, n4 list: python tools/flow_tps.py 128,256"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_14417_b200 as moe  # noqa: E402

prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
tag = f"MOE_FUSED={os.environ.get('MOE_FUSED', 'flow')} MOE_BAR_MODE={os.environ.get('MOE_BAR_MODE', '0')}"
for n4 in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "128,256").split(",")]:
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(32, 8, 2, 4096, 14336, plan, max_tokens=1, seed=0, norm_eps=1e-5)
    eng.synth_input(0, 1)
    eng.decode(1)
    eng.sync()
    ms = bench.time_engine(moe, torch, eng, 1, 80, 3)
    print(f"{tag} n4={n4:3d} {1000 / ms:7.1f} tok/s", flush=True)
    eng.close()
