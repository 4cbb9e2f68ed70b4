import sys, time, threading, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2407_14417_b200 as moe
sys.path.insert(0, 'tests')
from test_gpu_ep_engine import quality_plan, engine, _DevBytes
from helpers import TINY
plan = quality_plan(moe, TINY, 8, 1)
G, T = 2, 1
TC = int(os.environ.get('TCMIN', '0')); DELAY = float(os.environ.get('DELAY', '0'))
engs = [engine(moe, TINY, plan, T, 5, 1e-5, r, G, graphs=False, tc_min=TC) for r in range(G)]
bases = [e.ep_buffer()[0] for e in engs]
print("bases", [hex(b) for b in bases], [e.ep_buffer()[1] for e in engs], flush=True)
for e in engs: e.ep_set_peers(bases)
errs = []
def go(e):
    time.sleep(DELAY * e.ep_rank)
    try:
        e.decode(T); print("enqueued", e.ep_rank, flush=True); e.sync(); print("synced", e.ep_rank, flush=True)
    except Exception as ex:
        errs.append(ex)
th = [threading.Thread(target=go, args=(e,)) for e in engs]
for t in th: t.start()
time.sleep(3)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for r, b in enumerate(bases):
        v = torch.as_tensor(_DevBytes(b + 8448, 64), device="cuda").to("cpu", non_blocking=False)
        print("rank", r, "flags", np.frombuffer(v.numpy().tobytes(), np.uint32)[:16], flush=True)
for t in th: t.join()
print("errs", errs)
