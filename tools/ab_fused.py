"""A/B of the batch-1 decode: the fused one-launch step (dataflow
decode_flow_kernel, grid-barrier decode_step_kernel) vs five launches per
layer (CUDA-event timed graph replays, 8 inputs), Mixtral shape, n4 sweep."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_14417_b200 as moe  # noqa: E402

prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
pts = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "0,128,256").split(",")]
for n4 in pts:
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
    row = {}
    for name in ("per-layer", "step", "flow"):
        os.environ["MOE_FUSED"] = name
        eng = moe.MoeEngine(32, 8, 2, 4096, 14336, plan, max_tokens=1, seed=0, norm_eps=1e-5,
                            per_layer_decode=name == "per-layer")
        eng.synth_input(0, 1)
        eng.decode(1)
        eng.sync()
        ms = bench.time_engine(moe, torch, eng, 1, 80, 3)
        extra = ""
        if name != "per-layer":
            fm, fb = eng.profile_fused()
            extra = f" (launch {fm:.4f} ms, {fb / fm / 1e6:.0f} GB/s)"
        row[name] = f"{1000 / ms:7.1f} tok/s{extra}"
        eng.close()
    print(f"n4={n4:3d}  " + "   ".join(f"{k} {v}" for k, v in row.items()), flush=True)
