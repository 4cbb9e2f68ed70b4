"""Debug: fused vs per-layer vs oracle on small configurations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_14417_b200 as moe  # noqa: E402
from oracle.oracle import OracleLib  # noqa: E402

orc = OracleLib()


def bf(a):
    return (a.astype(np.uint32) << 16).view(np.float32)


for L, prec_mix, eps in [(1, [0] * 8, 0.0), (1, [1] * 8, 0.0), (1, [0, 1] * 4, 0.0), (1, [0] * 8, 1e-5)]:
    d, f = 512, 1792
    prof = moe.profile_for_shape(d, f, L, 8, 2)
    plan = moe.assign_locations(prec_mix * L, moe.HardwareProfile(10**15), prof)
    outs = []
    for per_layer in (False, True):
        eng = moe.MoeEngine(L, 8, 2, d, f, plan, max_tokens=1, seed=42, norm_eps=eps, per_layer_decode=per_layer)
        eng.synth_input(0, 1)
        eng.decode(1)
        eng.sync()
        t = torch.as_tensor(type("B", (), {"__cuda_array_interface__": {"shape": (d * 2,), "typestr": "|u1",
                                                                          "data": (eng.output_ptr, False),
                                                                          "version": 3}})(), device="cuda")
        outs.append(t.cpu().numpy().view(np.uint16).copy())
        rt = eng.last_routing(1)
        eng.close()
    m = orc.model(L, 8, 2, d, f, 42, eps)
    x = orc.step_input(m, 0, 1)
    for l in range(L):
        x, idx, _, _ = orc.moe_layer(m, l, prec_mix, x, 1)
    ref = bf(x.reshape(-1))
    a, b = bf(outs[0]), bf(outs[1])
    print(f"L={L} prec={prec_mix[:2]} eps={eps}: fused-vs-perlayer max {np.abs(a - b).max():.3e} "
          f"(n diff {(outs[0] != outs[1]).sum()}), fused-vs-oracle {np.abs(a - ref).max():.3e}, "
          f"perlayer-vs-oracle {np.abs(b - ref).max():.3e}, |ref| {np.abs(ref).max():.3e}, routing {rt} oracle {idx}")
