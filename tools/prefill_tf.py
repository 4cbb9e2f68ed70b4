"""tcgen05 prefill TFLOP/s (one Mixtral layer, bench.py's prefill measurement):
python tools/prefill_tf.py [T list]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2407_14417_b200 as moe  # noqa: E402

pts = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048,4096").split(",")]
prof1 = moe.profile_for_shape(bench.D_MODEL, bench.D_FFN, 1, bench.EXPERTS, bench.TOPK)
for prec in [int(p) for p in os.environ.get("PREC", "1,0").split(",")]:
    plan1 = moe.assign_locations([prec] * bench.EXPERTS, moe.HardwareProfile(10**15), prof1)
    eng = moe.MoeEngine(1, bench.EXPERTS, bench.TOPK, bench.D_MODEL, bench.D_FFN, plan1, max_tokens=max(pts), seed=0,
                        norm_eps=bench.NORM_EPS)
    for tp in pts:
        eng.synth_input(1, tp)
        eng.decode(tp)
        eng.sync()
        fm = sorted(eng.profile_step(tp)[0][0] for _ in range(5))
        ffn = fm[2]
        tf = 6.0 * bench.D_MODEL * bench.D_FFN * tp * bench.TOPK / (ffn * 1e-3) / 1e12
        print(f"{'bf16' if prec else 'int4'} T={tp:5d} {ffn:7.4f} ms {tf:7.1f} TF/s", flush=True)
    eng.close()
