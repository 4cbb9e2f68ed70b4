"""Phase timeline of the fused batch-1 decode step (decode_flow_kernel, or
decode_step_kernel with MOE_FUSED=step):
per layer, globaltimer stamps of every CTA at the phase boundaries, reported
as min / median / max over CTAs relative to the layer's first stamp,
averaged over the layers.  usage: python tools/trace_fused.py [n4] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_14417_b200 as moe  # noqa: E402

n4 = int(sys.argv[1]) if len(sys.argv) > 1 else 256
L = 32
prof = moe.profile_for_shape(4096, 14336, L, 8, 2)
plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(L, 8, 2, 4096, 14336, plan, max_tokens=1, seed=0, norm_eps=1e-5)
sms = torch.cuda.get_device_properties(0).multi_processor_count
S = 18
FLOW = os.environ.get("MOE_FUSED", "flow") != "step"
names = ["layer start", "routing done", "gate/up done", "after bar 1", "swiglu done", "after bar 2", "h resident",
         "down done", "after bar 3", "combine done", "r: x loaded", "r: rstd", "r: normalised", "r: logits",
         "r: topk+rows", "r: w0 topk+perm", "r: w1 rows"]
buf = torch.zeros(L * sms * S, dtype=torch.int64, device="cuda")
eng.synth_input(0, 1)
for _ in range(5):
    eng.decode(1)
eng.sync()
acc = []
for rep in range(5):
    for _ in range(10):
        eng.decode(1)
    eng.sync()
    moe.lib().moe_debug_fused_trace(buf.data_ptr())
    eng.decode(1)
    eng.sync()
    moe.lib().moe_debug_fused_trace(None)
    tr = buf.cpu().numpy().reshape(L, sms, S).astype(np.float64)
    acc.append(tr)
tr = np.median(np.stack(acc), axis=0)  # [L][sms][S]
MHZ = float(os.environ.get("SM_MHZ", "1965"))  # stamps are SM cycles (clock64), per CTA
# us from the layer's earliest CTA start (SM clocks are not synchronised across SMs, but
# clock64 counts from a common reset closely enough at this scale; ABS=0 -> per-CTA start)
if FLOW and os.environ.get("ABS", "1") == "1":
    # flow kernel: every CTA leaves its x-ready wait within ~1 round trip of the others (one
    # counter), so each CTA's stamps are taken relative to its own x-ready of the layer; the
    # previous layer's tail shows up as the layer period
    rel = (tr - tr[:, :, 1:2]) / MHZ
else:
    rel = (tr - tr[:, :, :1]) / MHZ  # us from this CTA's own layer start
print(f"== fused step ({'flow' if FLOW else 'step'}), n4={n4}: phase stamps (us from each CTA's layer start, SM clock; avg over {L} layers) "
      f"min / median / max over {sms} CTAs")
order = [0, 10, 11, 12, 13, 15, 16, 14, 1, 2, 3, 4, 5, 6, 7, 8, 9]
if FLOW:  # decode_flow_kernel's stamps (warp 0, finisher warp at 7)
    names[:16] = ["layer start", "x ready", "logits", "routing done", "w0 first down", "w0 items done",
                  "-", "finisher done", "fin: last unit rel", "fin: chunks in", "fin: last tile data",
                  "fin: last tile rel", "t0: xdone seen", "fin: last unit data", "-", "last warp done"]
    order = [1, 2, 3, 13, 8, 9, 4, 5, 15, 10, 11, 7]
for i in order:
    n = names[i]
    v = rel[:, :, i]
    print(f"   {n:14s} {v.min(axis=1).mean():7.2f} {np.median(v, axis=1).mean():7.2f} {v.max(axis=1).mean():7.2f}")
span = np.median(tr[1:, :, 1 if FLOW else 0] - tr[:-1, :, 1 if FLOW else 0], axis=1) / MHZ
print(f"   layer period   {span.mean():7.2f} us (median over CTAs)")
