"""Kernel timeline of one Mixtral-shaped MoE layer decode step (CUDA graph,
batch T): per kernel the first entry, first post-PDL-wait and last end,
relative to the route kernel's entry.
usage: python tools/trace_layer.py [precision 0|1] [T] [graphs 0|1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_14417_b200 as moe

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
graphs = bool(int(sys.argv[3])) if len(sys.argv) > 3 else True
L, E, k, d, f = 1, 8, 2, 4096, 14336
prof = moe.profile_for_shape(d, f, L, E, k)
plan = moe.assign_locations([prec] * (L * E), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(L, E, k, d, f, plan, max_tokens=T, use_graphs=graphs)
names = ["route", "route: x staged | logits | topk+xperm", "gate/up stream", "swiglu finalize", "down stream", "out finalize"]
buf = torch.zeros(6 * 3, dtype=torch.int64, device="cuda")
eng.synth_input(0, T)
for _ in range(5):
    eng.decode(T)
eng.sync()
res = []
for rep in range(5):
    init = np.zeros((6, 3), dtype=np.uint64)
    init[:, 0] = init[:, 1] = np.iinfo(np.uint64).max
    buf.copy_(torch.from_numpy(init.view(np.int64).reshape(-1)))
    torch.cuda.synchronize()
    for _ in range(20):          # keep the GPU busy and clocked up
        eng.decode(T)
    moe.lib().moe_debug_layer_trace(buf.data_ptr(), eng.stream_ptr)
    eng.decode(T)
    moe.lib().moe_debug_layer_trace(None, eng.stream_ptr)
    eng.sync()
    res.append(buf.cpu().numpy().view(np.uint64).reshape(6, 3).astype(np.float64))
tr = np.median(np.stack(res), axis=0)
t0 = tr[0, 0]
print(f"== one layer, {'bf16' if prec else 'int4'} experts, T={T}, graphs={graphs} (us from route entry; median of 5)")
for i, n in enumerate(names):
    e, w, x = (tr[i] - t0) / 1e3
    if i == 1:
        print(f"   {n:16s} {e:7.1f} {w:7.1f} {x:7.1f}")
        continue
    print(f"   {n:16s} entry {e:7.1f}  wait-done {w:7.1f}  end {x:7.1f}   (run {x - w:6.1f})")
print(f"   layer span {(tr[5, 2] - t0) / 1e3:.1f} us")
