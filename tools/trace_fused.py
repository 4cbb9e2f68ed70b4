"""Phase timeline of the fused batch-1 decode step (decode_step_kernel):
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
S = 10
names = ["layer start", "routing done", "gate/up done", "after bar 1", "swiglu done", "after bar 2", "h resident",
         "down done", "after bar 3", "combine done"]
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
rel = (tr - tr[:, :, :1].min(axis=1, keepdims=True)) / 1e3  # us from the layer's first start
print(f"== fused step, n4={n4}: phase stamps (us from the layer's earliest start; avg over {L} layers) "
      f"min / median / max over {sms} CTAs")
for i, n in enumerate(names):
    v = rel[:, :, i]
    print(f"   {n:14s} {v.min(axis=1).mean():7.2f} {np.median(v, axis=1).mean():7.2f} {v.max(axis=1).mean():7.2f}")
span = (tr[1:, :, 0].min(axis=1) - tr[:-1, :, 0].min(axis=1)) / 1e3
print(f"   layer period   {span.mean():7.2f} us  (step {(tr[-1, :, 9].max() - tr[0, :, 0].min()) / 1e3:.1f} us)")
