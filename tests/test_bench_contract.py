"""bench.py's JSON contract on the CPU side: the reference arm (the oracle
port timed on host threads) prints one line with the keys the driver reads,
and the Pareto tool's unmeasured table carries the reference schema."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    """--impl reference at the tiny shape: the CPU port through the whole
    stack per step, plan from the reference's planner, and the product
    library never loaded (the arm loaded libmoe_b200.so)."""
    probe = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--shape', 'tiny', '--n4', '8', "
             "'--steps', '16', '--warmup', '3']; runpy.run_path('bench.py', run_name='__main__'); "
             "maps = open('/proc/self/maps').read(); "
             "print('LOADED_PRODUCT' if 'libmoe_b200' in maps else 'PRODUCT_NOT_LOADED', file=sys.stderr)")
    r = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("port", "reference")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "PRODUCT_NOT_LOADED" in r.stderr
    assert d["steps"] == 16 and abs(d["ms_per_step"] * 16 / 1e3 - 16 / d["value"]) < 1e-3
    assert d["config"]["layers"] == 2 and "make_plan" in d["plan_source"]


def test_golden_plans_equal_ours(moe):
    """The reference planner's frozen Mixtral plans (the reference arm's
    fallback) equal this library's make_plan."""
    with open(os.path.join(ROOT, "tests", "golden", "mixtral_plans.json")) as fh:
        plans = json.load(fh)["plans"]
    prof = moe.profile_for_shape(4096, 14336, 32, 8, 2)
    for n4, prec in plans.items():
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, int(n4), 0), moe.HardwareProfile(10**15), prof)
        assert plan.precision == prec, n4


def test_gemv_max_tokens(moe):
    """the exported limit follows the segment-table bound
    min(E, T*k) + ceil(T*k/8) <= 64."""
    lim = moe.lib().moe_gemv_max_tokens
    for E, k in [(8, 2), (16, 4), (64, 8), (64, 2), (2, 1)]:
        T = lim(E, k)
        seg = lambda t: min(E, t * k) + -(-t * k // 8)  # noqa: E731
        assert seg(T) <= 64 < seg(T + 1)
    assert lim(8, 2) >= 31  # the engine's GEMV range below tc_min_tokens = 32


def test_pareto_tool_unmeasured_table():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "pareto_sweep.py"), "--no-measure",
                        "--mem-range", "24GB:48GB:24GB", "--n4-grid", "0,256"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[0] == ("budget_bytes,n4,n_gpu,gpu_bytes,throughput_tps,hit_rate,bytes_transferred,ppl_estimate,"
                        "on_frontier,status")
    assert len(lines) == 5 and all(l.endswith(",ok") for l in lines[1:])
