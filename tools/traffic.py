"""ncu DRAM traffic of the expert-FFN launches of one profiled decode step
(the bench's roofline configuration) -> profiles/r02_traffic.json.

Usage (on the GPU box):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --profile-from-start off --clock-control none --csv --log-file gpurun_out/traffic.csv \
      python tools/traffic.py run
  python tools/traffic.py summarize gpurun_out/traffic.csv gpurun_out/traffic_alg.json > profiles/r02_traffic.json

`run` builds the bench engine (n4, batch T), warms it, then runs exactly one
profile_step on input bench.TRAFFIC_INPUT between cudaProfilerStart/Stop and
writes that step's per-layer algorithmic bytes next to the ncu log.
"""
import csv
import json
import os
import subprocess
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
    eng = moe.MoeEngine(bench.LAYERS, bench.EXPERTS, bench.TOPK, bench.D_MODEL, bench.D_FFN, plan, max_tokens=T,
                        seed=0, norm_eps=bench.NORM_EPS)
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.profile_step(T)  # warm (geometry caches, first-touch)
    eng.synth_input(bench.TRAFFIC_INPUT, T)
    eng.sync()
    torch.cuda.profiler.start()
    _, fb, _ = eng.profile_step(T)
    torch.cuda.profiler.stop()
    eng.close()
    with open(os.path.join(ROOT, out), "w") as fh:
        json.dump({"n4": n4, "tokens": T, "input": bench.TRAFFIC_INPUT, "layers": bench.LAYERS,
                   "algorithmic_bytes_per_layer": round(sum(fb) / len(fb)), "algorithmic_bytes": fb}, fh)


def summarize(csv_path, alg_path):
    with open(alg_path) as fh:
        alg = json.load(fh)
    rows = []
    with open(csv_path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        rows.append(r)
    per = {}
    for r in rows:
        name = r["Kernel Name"]
        if not any(k in name for k in FFN_KERNELS):
            continue
        key = (r["ID"], name)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        per.setdefault(key, {})[r["Metric Name"]] = v * scale
    dram = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in per.values())
    launches = len(per)
    head = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True, cwd=ROOT).stdout.strip()
    print(json.dumps({"n4": alg["n4"], "tokens": alg["tokens"], "input": alg["input"], "layers": alg["layers"],
                      "ffn_launches": launches, "dram_bytes_step": round(dram),
                      "dram_bytes_per_layer": round(dram / alg["layers"]),
                      "algorithmic_bytes_per_layer": alg["algorithmic_bytes_per_layer"],
                      "ratio": round(dram / alg["layers"] / alg["algorithmic_bytes_per_layer"], 4),
                      "kernels": FFN_KERNELS, "commit": head,
                      "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one profile_step "
                             "(tools/traffic.py)"}, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(*(int(v) for v in sys.argv[2:4]))
    else:
        summarize(sys.argv[2], sys.argv[3])
