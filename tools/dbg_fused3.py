"""Debug: compare the GEMV workspace intermediates of the fused and per-layer paths."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_14417_b200 as moe  # noqa: E402


def grab(eng, which):
    p, n = C.c_void_p(), C.c_size_t()
    assert moe.lib().moe_debug_engine_buffer(eng._h, which, C.byref(p), C.byref(n)) == 0
    t = torch.as_tensor(type("B", (), {"__cuda_array_interface__": {"shape": (n.value,), "typestr": "|u1",
                                                                      "data": (p.value, False), "version": 3}})(),
                        device="cuda")
    return t.cpu().numpy().copy()


L, d, f = 1, 512, 1792
prof = moe.profile_for_shape(d, f, L, 8, 2)
plan = moe.assign_locations([0] * 8, moe.HardwareProfile(10**15), prof)
bufs = {}
for per_layer in (False, True):
    eng = moe.MoeEngine(L, 8, 2, d, f, plan, max_tokens=1, seed=42, norm_eps=1e-5, per_layer_decode=per_layer)
    eng.synth_input(0, 1)
    eng.decode(1)
    eng.sync()
    bufs[per_layer] = [grab(eng, w) for w in range(5)]
    eng.close()
names = ["part0", "part1", "hperm", "hperm16", "hsum"]
G0, G1 = d // 128, f // 128
for w, n in enumerate(names):
    a, b = bufs[False][w], bufs[True][w]
    if w in (0, 1):
        a, b = a.view(np.float32), b.view(np.float32)
    elif w == 4:
        a, b = a.view(np.float32), b.view(np.float32)
    else:
        a, b = a.view(np.uint16), b.view(np.uint16)
    # only the regions the T=1 step writes
    if w == 0:
        a, b = a[:G0 * 2 * 2 * f], b[:G0 * 2 * 2 * f]
    if w == 1:
        a, b = a[:G1 * 2 * d], b[:G1 * 2 * d]
    diff = np.nonzero(a != b)[0]
    print(f"{n}: {len(diff)} of {a.size} differ; first {diff[:10]}; vals fused {a[diff[:4]]} per-layer {b[diff[:4]]}")
