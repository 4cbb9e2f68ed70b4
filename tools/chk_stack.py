"""Decode one token through the Mixtral-shaped stack layer by layer and print
per-layer routing and activation magnitude (debug)."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2407_14417_b200 as moe
n4 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
L, E, k, d, f = 32, 8, 2, 4096, 14336
prof = moe.profile_for_shape(d, f, L, E, k)
plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(L, E, k, d, f, plan, max_tokens=1, seed=0, use_graphs=False)
eng.synth_input(7, 1); eng.sync()
x = torch.empty(d, dtype=torch.int16, device='cuda')
x.copy_(torch.as_tensor(np.zeros(d, np.int16)))
import ctypes
src = torch.zeros(d, dtype=torch.int16, device='cuda')
ptr = eng.input_ptr
class _D:
    def __init__(s, p, n): s.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (p, False), "version": 3}
src.copy_(torch.as_tensor(_D(ptr, d), device='cuda'))
out = torch.empty(d, dtype=torch.int16, device='cuda'); idx = torch.empty(k, dtype=torch.int32, device='cuda')
w = torch.empty(k, dtype=torch.float32, device='cuda'); lg = torch.empty(E, dtype=torch.float32, device='cuda')
for l in range(L):
    eng.forward_layer(l, src, 1, out, idx, w, lg); eng.sync()
    v = (out.cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    print(l, idx.cpu().numpy(), 'maxabs %.3e' % np.abs(v).max(), 'nan', np.isnan(v).sum(), 'lg', np.round(lg.cpu().numpy(), 2)[:4])
    src = out.clone()
