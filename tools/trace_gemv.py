"""Per-warp phase timeline of the GEMV passes of one Mixtral-shaped layer.
usage: python tools/trace_gemv.py [precision 0|1] [T]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_14417_b200 as moe

prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L, E, k, d, f = 4, 8, 2, 4096, 14336
prof = moe.profile_for_shape(d, f, L, E, k)
plan = moe.assign_locations([prec] * (L * E), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(L, E, k, d, f, plan, max_tokens=T, use_graphs=False)
W = 148 * int(os.environ.get('GEMV_WARPS', '8'))
buf = torch.zeros(2 * W * 8, dtype=torch.int64, device="cuda")
eng.synth_input(0, T)
for _ in range(3):
    eng.decode(T)
eng.sync()
moe.lib().moe_debug_gemv_trace(buf.data_ptr())
eng.decode(T)
eng.sync()
moe.lib().moe_debug_gemv_trace(None)
tr = buf.view(2, W, 8).cpu().numpy()
for p, name in enumerate(["gate/up stream", "down stream"]):
    t = tr[p]
    live = t[:, 3] > 0
    t = t[live]
    t0 = t[:, 0].min()
    items = t[:, 4] & 0xffffffff
    runs = t[:, 4] >> 32
    print(f"== {name} ({'bf16' if prec else 'int4'}, T={T}) warps={len(t)} items={items.sum()} runs={runs.sum()}")
    for lab, col in (("mbar wait", 7),):
        v = t[:, col] / 1e3
        print(f"   {lab:10s} per warp: med {np.median(v):6.1f}  p90 {np.percentile(v,90):6.1f}  max {v.max():6.1f} us")
    span = (t[:, 3].max() - t0) / 1e3
    print(f"   span {span:.1f} us  entry spread {(t[:,0].max()-t0)/1e3:.1f} us")
    for lab, a, b in (("entry->wait", 0, 1), ("wait->item0", 1, 2), ("item0->end", 2, 3)):
        v = (t[:, b] - t[:, a]) / 1e3
        print(f"   {lab:12s} min {v.min():6.1f}  med {np.median(v):6.1f}  max {v.max():6.1f} us")
    ends = (t[:, 3] - t0) / 1e3
    print(f"   end times  p10 {np.percentile(ends,10):.1f}  p50 {np.percentile(ends,50):.1f}  p90 {np.percentile(ends,90):.1f}  max {ends.max():.1f} us")
