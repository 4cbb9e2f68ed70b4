"""bench.py's JSON contract on the CPU side: the reference arm (the oracle
port timed on host threads) prints one line with the keys the driver reads,
and the Pareto tool's unmeasured table carries the reference schema."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_pareto_tool_unmeasured_table():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pareto_sweep.py"), "--no-measure",
                        "--mem-range", "24GB:48GB:24GB", "--n4-grid", "0,256"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[0] == ("budget_bytes,n4,n_gpu,gpu_bytes,throughput_tps,hit_rate,bytes_transferred,ppl_estimate,"
                        "on_frontier,status")
    assert len(lines) == 5 and all(l.endswith(",ok") for l in lines[1:])
