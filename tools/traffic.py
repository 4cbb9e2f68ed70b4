"""ncu DRAM traffic of the bench's roofline kernels -> profiles/r02_traffic.json.

Two captures at the headline configuration (n4, batch T, input bench.TRAFFIC_INPUT):
  fused      one fused-step launch (decode_flow_kernel: the whole batch-1 step)
  per_layer  the expert-FFN launches (stream_kernel x2, finalize_h, finalize_out)
             of one per-layer-kernel step, summed and divided by the layers

Usage (on the GPU box):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --profile-from-start off --clock-control none --csv --log-file gpurun_out/traffic.csv \
      python tools/traffic.py run
  python tools/traffic.py summarize gpurun_out/traffic.csv gpurun_out/traffic_alg.json > profiles/r02_traffic.json
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FFN_KERNELS = ("stream_kernel", "finalize_h_kernel", "finalize_out_kernel")


def run(n4=128, T=1, out="gpurun_out/traffic_alg.json"):
    import torch

    import bench
    import paper_2407_14417_b200 as moe
    prof = moe.profile_for_shape(bench.D_MODEL, bench.D_FFN, bench.LAYERS, bench.EXPERTS, bench.TOPK)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
    res = {"n4": n4, "tokens": T, "input": bench.TRAFFIC_INPUT, "layers": bench.LAYERS}
    # capture 1: the fused step
    eng = moe.MoeEngine(bench.LAYERS, bench.EXPERTS, bench.TOPK, bench.D_MODEL, bench.D_FFN, plan, max_tokens=T,
                        seed=0, norm_eps=bench.NORM_EPS)
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.profile_fused()
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.sync()
    torch.cuda.profiler.start()
    _, fb = eng.profile_fused()
    torch.cuda.profiler.stop()
    eng.close()
    res["fused_algorithmic_bytes"] = fb
    # capture 2: the per-layer kernels
    eng = moe.MoeEngine(bench.LAYERS, bench.EXPERTS, bench.TOPK, bench.D_MODEL, bench.D_FFN, plan, max_tokens=T,
                        seed=0, norm_eps=bench.NORM_EPS, per_layer_decode=True)
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.profile_step(T)
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.sync()
    torch.cuda.profiler.start()
    _, lb, _ = eng.profile_step(T)
    torch.cuda.profiler.stop()
    eng.close()
    res["per_layer_algorithmic_bytes"] = round(sum(lb) / len(lb))
    with open(os.path.join(ROOT, out), "w") as fh:
        json.dump(res, fh)


def summarize(csv_path, alg_path, commit=""):
    with open(alg_path) as fh:
        alg = json.load(fh)
    with open(csv_path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    per = {}
    for r in csv.DictReader(lines):
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(r["Metric Unit"], 1)
        per.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = v * scale

    def dram(m):
        return m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)

    fused = [(n, m) for (i, n), m in per.items() if "decode_flow_kernel" in n or "decode_step_kernel" in n]
    ffn = [m for (i, n), m in per.items() if any(k in n for k in FFN_KERNELS)]
    base = {"n4": alg["n4"], "tokens": alg["tokens"], "input": alg["input"], "commit": commit}
    out = {"how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (tools/traffic.py)"}
    if fused:
        name, m = fused[0]
        kname = "decode_flow_kernel" if "decode_flow_kernel" in name else "decode_step_kernel"
        out["fused"] = dict(base, what="one %s launch (whole %d-layer step)" % (kname, alg["layers"]),
                            dram_bytes=round(dram(m)), algorithmic_bytes=alg["fused_algorithmic_bytes"],
                            ratio=round(dram(m) / alg["fused_algorithmic_bytes"], 4),
                            ncu_time_us=round(m.get("gpu__time_duration.sum", 0) / 1e3, 1))
    if ffn:
        tot = sum(dram(m) for m in ffn)
        out["per_layer"] = dict(base, what="the expert-FFN launches of one per-layer step, per layer (%d launches / "
                                           "%d layers)" % (len(ffn), alg["layers"]),
                                dram_bytes=round(tot / alg["layers"]), algorithmic_bytes=alg["per_layer_algorithmic_bytes"],
                                ratio=round(tot / alg["layers"] / alg["per_layer_algorithmic_bytes"], 4))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(*(int(v) for v in sys.argv[2:4]))
    else:
        summarize(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
