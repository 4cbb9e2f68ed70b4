"""Debug: determinism of the fused and per-layer batch-1 paths."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_14417_b200 as moe  # noqa: E402


def out(eng, n):
    t = torch.as_tensor(type("B", (), {"__cuda_array_interface__": {"shape": (n,), "typestr": "|u1",
                                                                      "data": (eng.output_ptr, False), "version": 3}})(),
                        device="cuda")
    return t.cpu().numpy().copy()


for (L, d, f, n4, eps) in [(2, 512, 1792, 8, 0.0), (2, 512, 1792, 8, 1e-5), (1, 512, 1792, 8, 1e-5)]:
    prof = moe.profile_for_shape(d, f, L, 8, 2)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 1), moe.HardwareProfile(10**15), prof)
    res = {}
    for per_layer in (False, True):
        for graphs in (True, False):
            eng = moe.MoeEngine(L, 8, 2, d, f, plan, max_tokens=1, seed=42, norm_eps=eps, per_layer_decode=per_layer,
                                use_graphs=graphs)
            outs = []
            for rep in range(30):
                eng.synth_input(rep % 3, 1)
                eng.decode(1)
                eng.sync()
                outs.append(out(eng, 2 * d))
            eng.close()
            res[(per_layer, graphs)] = outs
    base = res[(True, True)]
    for key, outs in res.items():
        nd = [int((o != base[i]).sum()) for i, o in enumerate(outs)]
        print(f"L={L} n4={n4} eps={eps} per_layer={key[0]} graphs={key[1]}: bytes differing vs per-layer graph run: {nd}")
