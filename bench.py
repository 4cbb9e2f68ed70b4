#!/usr/bin/env python
"""bench.py -- decode tokens/s of the Mixtral-8x7B-shaped MoE expert-layer
stack vs the number of 4-bit experts (BASELINE.json metric), on B200.

Workload (BASELINE.json configs[2], the metric's "decode tokens/s vs #4-bit
experts" on one GPU): 32 layers x 8 experts (d=4096, ffn=14336), top-2,
batch-1 decode, synthetic weights from the seeded generator, plan =
plan_quality(n4, seed 0) with every expert device-resident.  The headline
`value` is at n4 = 128 of 256 (half the experts int4-g128); `sweep` carries
the full n4 = 0..256 curve.  A "step" = one decode token through all 32
layers (route -> gate/up GEMV -> down GEMV -> combine, one CUDA graph).

  value     device-timed (CUDA events on the engine stream), inputs resident
  e2e       through the public API with host buffers (moe_engine_decode_host:
            H2D of the token's embedding, decode, D2H of the output, synced)
  roofline  the dominant kernel pair (expert FFN gate/up + down) timed with
            CUDA events per layer on its launch stream; algorithmic bytes =
            distinct selected experts' weights+scales + activations
  cpu_baseline  the CPU port (oracle/, OpenMP over all host threads) on a
            bounded sample: one token input through the full 32-layer stack
            (its selected experts materialised, untimed), repeated

No L2 flush is needed: one step streams 64 distinct experts (5.8-22.5 GB)
through a 126 MB L2.  `--impl reference` times the reference path on the
host: the reference (/root/reference) has no tensor math, so
its arm is the CPU port of this path (oracle/, OpenMP over every host
thread) driven by the reference's own planner (oracle/_ref make_plan) --
the whole 32-layer stack per step, never the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D_MODEL, D_FFN, LAYERS, EXPERTS, TOPK = 4096, 14336, 32, 8, 2
# Mixtral decoder layers apply post_attention_layernorm (RMSNorm, eps 1e-5)
# before the MoE block; without it the synthetic residual stream overflows
# after ~12 layers and the routing degenerates (tests: prenorm stack test).
NORM_EPS = 1e-5
METRIC = "decode tokens/s vs #4-bit experts (Mixtral-8x7B shape); expert-FFN HBM GB/s"


TRAFFIC_INPUT = 7  # the token input profile_step runs for the roofline (and tools/traffic.py under ncu)


def _traffic(n4, T, alg_bytes, fused=False):
    """ncu dram read+write of the dominant launch(es), captured by
    tools/traffic.py for this configuration and input (profiles/r02_traffic.json),
    next to the algorithmic bytes of the same step; null when absent or when
    the recorded algorithmic bytes disagree (another kernel or routing).
    fused: per launch of the fused step kernel (one step); else per layer of the
    expert-FFN launches."""
    path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
    except Exception:
        return None, "no ncu traffic capture for this configuration"
    key = "fused" if fused else "per_layer"
    t = t.get(key, t if not fused else None)
    if not t or (t.get("n4"), t.get("tokens"), t.get("input")) != (n4, T, TRAFFIC_INPUT) or \
            int(t["algorithmic_bytes"]) != int(alg_bytes):
        return None, "profiles/r02_traffic.json has no capture of this kernel / configuration"
    return int(t["dram_bytes"]), ("ncu dram__bytes_read+write of %s on input %d (profiles/r02_traffic.json, "
                                  "commit %s); algorithmic %d B" % (t["what"], TRAFFIC_INPUT, t.get("commit", "?"),
                                                                    int(t["algorithmic_bytes"])))


def _peak_tflops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["bf16_tflops"])
    except Exception:
        return 1590.0


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled every 10 ms through NVML on a
    background thread during the timed region (nvidia-smi's 100 ms floor
    missed short regions); one sample is always taken at exit."""

    PERIOD_S = 0.010
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.err = None
        self._stop = None
        self._thr = None

    def _sample(self, nv, h):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((sm, mx, r))

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis and vis.split(",")[self.dev].isdigit() else self.dev
            h = nv.nvmlDeviceGetHandleByIndex(idx)
        except Exception as exc:  # no NVML: report it, never fake a clock
            self.err = f"nvml unavailable: {exc}"
            return self
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self._sample(nv, h)
                except Exception as exc:
                    self.err = str(exc)
                    return
                self._stop.wait(self.PERIOD_S)
            self._sample(nv, h)

        self._thr = threading.Thread(target=run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        if self._thr is not None:
            self._stop.set()
            self._thr.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"], "samples": 0}
        reasons = sorted({n for _, _, r in self.rows for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "period_ms": self.PERIOD_S * 1e3,
                "source": "NVML (nvmlDeviceGetClockInfo / CurrentClocksEventReasons)"}


N_INPUTS = 8  # distinct token inputs per timing: the routing (and so the bytes) varies per input


def bench_config(args, T, world, parallelism=None):
    """The workload description both arms print (identical keys and values)."""
    return {"workload": "mixtral8x7b-shape 32-layer MoE stack, batch-%d decode" % T, "n4": args.n4,
            "layer": "x + MoE(RMSNorm(x)) (decoder-layer norm eps 1e-5, unit weight; no attention)",
            "of": LAYERS * EXPERTS, "plan": "plan_quality seed 0, all device-resident",
            "d_model": D_MODEL, "d_ffn": D_FFN, "layers": LAYERS, "experts": EXPERTS, "top_k": TOPK,
            "batch": T, "parallelism": parallelism or ("single" if world == 1 else "replicas"),
            "inputs": "%d distinct synthetic token inputs (1000..%d), steps split evenly over them (the routing, "
                      "hence the expert bytes per step, varies with the input)" % (N_INPUTS, 1000 + N_INPUTS - 1),
            "l2": "no flush: each step streams 5.8-22.5 GB of distinct expert weights >> 126 MB L2"}


def reference_plan_precision(n4):
    """plan_quality(n4, seed 0) precisions from the reference's own planner
    (oracle/_ref: /root/reference/proj/src/planner.cpp make_plan), falling
    back to the frozen reference output in tests/golden/mixtral_plans.json."""
    try:
        from oracle.oracle import RefLib, RefProfile
        ref = RefLib()
        prof = RefProfile(LAYERS, EXPERTS, TOPK, 0, 1, 6 * D_MODEL * D_FFN, 128.0 / 33.0, 1e-3, 1.0, 0.0)
        st, prec, loc, _ = ref.make_plan(prof, 10**15, 12.285e9, 1, n4, 0)  # 1 = Quality
        if st != 0:
            raise RuntimeError(ref.err())
        return [int(v) for v in prec], "oracle/_ref make_plan (the reference's planner)"
    except (FileNotFoundError, OSError):
        with open(os.path.join(ROOT, "tests", "golden", "mixtral_plans.json")) as fh:
            return json.load(fh)["plans"][str(n4)], "tests/golden/mixtral_plans.json (reference make_plan output)"


class CpuStack:
    """The 32-layer stack on the CPU port (oracle/, OpenMP): layer = x +
    MoE(RMSNorm(x)); experts are materialised on first use (untimed when
    `prepare` runs them first) and kept."""

    def __init__(self, precision, seed=0):
        from oracle.oracle import OracleLib, OrcExpert, _np_ptr
        self.orc = OracleLib()
        self.m = self.orc.model(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, seed, NORM_EPS)
        self.prec = precision
        self.wg = [self.orc.router_weights(self.m, l) for l in range(LAYERS)]
        self.arr = [(OrcExpert * EXPERTS)() for _ in range(LAYERS)]
        for l in range(LAYERS):
            for s_ in range(EXPERTS):
                self.arr[l][s_].precision = precision[l * EXPERTS + s_]
        self.keep = {}
        self._ptr = _np_ptr
        self.built = 0

    def _ensure(self, l, slots):
        for s_ in slots:
            e = l * EXPERTS + int(s_)
            if e in self.keep:
                continue
            a = self.arr[l][int(s_)]
            if self.prec[e] == 1:
                gu, dn = self.orc.expert_bf16(self.m, e)
                self.keep[e] = (gu, dn)
                a.w_gate_up, a.w_down = self._ptr(gu), self._ptr(dn)
            else:
                qgu, sgu, qd, sd = self.orc.expert_int4(self.m, e)
                self.keep[e] = (qgu, sgu, qd, sd)
                a.w_gate_up, a.s_gate_up, a.w_down, a.s_down = (self._ptr(v) for v in (qgu, sgu, qd, sd))
            self.built += 1

    def step(self, x, T, prepare=False):
        for l in range(LAYERS):
            if prepare:  # routing first, then the selected experts (untimed pass)
                xn = self.orc.rmsnorm(x, T, D_MODEL, NORM_EPS)
                idx, _, _ = self.orc.gate_topk(xn, self.wg[l], T, D_MODEL, EXPERTS, TOPK)
                self._ensure(l, set(idx.reshape(-1).tolist()))
            x, _ = self.orc.moe_layer_w(self.m, (self.wg[l], self.arr[l], None), x, T)
        return x

    def threads(self):
        return self.orc.num_threads()


def cpu_port_tokens_per_s(precision, T, seconds=12.0):
    """cpu_baseline: one token input (1000) through the full 32-layer stack on
    the CPU port; its selected experts materialised first (untimed), then
    repeated for ~`seconds`.  Returns (tok/s, threads, sample)."""
    stack = CpuStack(precision)
    x0 = stack.orc.step_input(stack.m, 1000, T)
    stack.step(x0, T, prepare=True)
    reps, t0 = 0, time.perf_counter()
    while True:
        stack.step(x0, T)
        reps += 1
        el = time.perf_counter() - t0
        if el >= seconds or reps >= 200:
            break
    tps = T * reps / el
    sample = (f"token input 1000 (batch {T}) through the full {LAYERS}-layer stack ({stack.built} selected experts "
              f"materialised untimed), {reps} repeats in {el:.1f} s")
    return tps, stack.threads(), sample


def run_reference(args, rank, world):
    """--impl reference: the reference path on the host's cores.  Rank 0 only
    (torchrun N > 1: the other ranks exit without work).  Never loads the
    product library."""
    if rank != 0:
        return
    T = args.tokens
    prec, plan_src = reference_plan_precision(args.n4)
    stack = CpuStack(prec)
    inputs = [stack.orc.step_input(stack.m, 1000 + i, T) for i in range(N_INPUTS)]
    t_prep = time.perf_counter()
    for x in inputs:  # materialise every expert the inputs route to (untimed)
        stack.step(x, T, prepare=True)
    t_prep = time.perf_counter() - t_prep
    for w in range(args.warmup):
        stack.step(inputs[w % N_INPUTS], T)
    per = [args.steps // N_INPUTS + (1 if i < args.steps % N_INPUTS else 0) for i in range(N_INPUTS)]
    t0 = time.perf_counter()
    for i in range(N_INPUTS):
        for _ in range(per[i]):
            stack.step(inputs[i], T)
    el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    tps = T * args.steps / el
    sample = (f"{args.steps} steps x batch {T} through the full {LAYERS}-layer stack, inputs 1000..{999 + N_INPUTS} "
              f"rotated as in the GPU arm ({stack.built} experts materialised untimed in {t_prep:.0f} s)")
    line = {"impl": "reference", "metric": METRIC, "value": round(tps, 4), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16 / int4-g128 weights, bf16 activations, fp32 accumulate",
            "data": "synthetic (seeded counter-based generator, int4 = RTN-g128 of the bf16 masters)",
            "config": bench_config(args, T, 1),
            "cpu_baseline": {"value": round(tps, 4), "unit": "tokens/s", "cores": stack.threads(), "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(tps, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "plan_source": plan_src,
            "note": "the reference has no tensor math (SPEC.md:13): its arm is the CPU port of this path "
                    "(oracle/, OpenMP over all host threads), driven by the reference's planner"}
    print(json.dumps(line), flush=True)




def time_engine(moe, torch, eng, T, steps, warmup, inputs=N_INPUTS):
    """ms per decode step, averaged over `inputs` different token inputs
    (steps/inputs back-to-back decodes of each, CUDA events on the engine
    stream around each run; the input write sits between the timed runs)."""
    stream = torch.cuda.ExternalStream(eng.stream_ptr)
    for w in range(warmup):
        eng.synth_input(w, T)
        eng.decode(T)
    eng.sync()
    inputs = max(1, min(inputs, steps))
    total, n = 0.0, 0
    for i in range(inputs):
        per = steps // inputs + (1 if i < steps % inputs else 0)  # exactly `steps` timed decodes in all
        eng.synth_input(1000 + i, T)
        eng.decode(T)  # first decode of this input (graph already captured) outside the timing
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(stream)
        for _ in range(per):
            eng.decode(T)
        end.record(stream)
        end.synchronize()
        total += start.elapsed_time(end)
        n += per
    return total / n


def run_ours(args, rank, world, device):
    import torch
    import paper_2407_14417_b200 as moe
    dist = None
    if world > 1:
        import torch.distributed as dist
    prof = moe.profile_for_shape(D_MODEL, D_FFN, LAYERS, EXPERTS, TOPK)
    T = args.tokens
    hbm_peak, peak_kind = peaks()
    s16, s4 = moe.expert_size(prof, 1), moe.expert_size(prof, 0)

    def build(n4):
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
        eng = moe.MoeEngine(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, plan, max_tokens=T, seed=args.seed + rank,
                            device=device, norm_eps=NORM_EPS)
        return plan, eng

    # ---- headline point ---------------------------------------------------
    plan, eng = build(args.n4)
    eng.synth_input(0, T)
    eng.decode(T)  # capture the graph
    eng.sync()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device) as clk:
        ms = time_engine(moe, torch, eng, T, args.steps, args.warmup)
    clocks = clk.summary()
    if dist:
        t = torch.tensor([ms], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * T * 1000.0 / ms

    # ---- roofline ------------------------------------------------------------
    # batch 1: the fused decode step is ONE launch (decode_flow_kernel) --
    # timed alone between CUDA events on the engine stream, against the
    # algorithmic bytes of the routing it made; otherwise the per-layer
    # expert FFN launches (gate/up stream + finalize_h + down stream +
    # finalize_out) bracketed per layer
    fused = eng.profile_fused() is not None
    if fused:
        runs = []
        for _ in range(5):
            eng.synth_input(TRAFFIC_INPUT, T)
            runs.append(eng.profile_fused())
        avg_ms = sorted(r[0] for r in runs)[len(runs) // 2]
        avg_bytes = runs[0][1]
        kps = 1
        ffn_share = avg_ms / ms
        traffic, traffic_note = _traffic(args.n4, T, avg_bytes, fused=True)
        kernel_desc = ("%s: the whole %d-layer batch-1 step in one cooperative launch (routing, "
                       "gate/up GEMV, SwiGLU, down GEMV, combine per layer%s), CUDA events on the engine stream; "
                       "median of 5 launches on input %d" % (
                           "decode_step_kernel" if os.environ.get("MOE_FUSED") == "step" else "decode_flow_kernel",
                           LAYERS, "" if os.environ.get("MOE_FUSED") == "step" else
                           "; dataflow hand-offs, no grid barriers inside a layer", TRAFFIC_INPUT))
    else:
        ffn_ms, ffn_bytes = [], []
        for _ in range(3):
            eng.synth_input(TRAFFIC_INPUT, T)
            m_, b_, kps = eng.profile_step(T)
            ffn_ms += m_
            ffn_bytes += b_
        traffic, traffic_note = _traffic(args.n4, T, round(sum(ffn_bytes[:LAYERS]) / LAYERS))
        avg_ms = sum(ffn_ms) / len(ffn_ms)
        avg_bytes = sum(ffn_bytes) / len(ffn_bytes)
        ffn_share = (avg_ms * LAYERS) / ms
        kernel_desc = ("expert FFN per layer: stream_kernel (gate/up) + finalize_h + stream_kernel (down) + "
                       "finalize_out, CUDA events on the engine stream")
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9

    # ---- e2e through the public API with host buffers -----------------------
    import numpy as np
    # N_INPUTS different pinned host inputs, rotated every step
    xhs = []
    for i in range(N_INPUTS):
        eng.synth_input(1000 + i, T)
        eng.sync()
        xh = torch.empty(T * D_MODEL, dtype=torch.int16).pin_memory()
        xh.copy_(torch.as_tensor(_DevBytes(eng.input_ptr, T * D_MODEL * 2), device=f"cuda:{device}").view(torch.int16).cpu())
        xhs.append(xh)
    oh = torch.empty(T * D_MODEL, dtype=torch.int16).pin_memory()
    for i in range(max(1, args.warmup)):
        eng.decode_host(xhs[i % N_INPUTS].data_ptr(), T, oh.data_ptr())
    e_steps = max(10, min(args.steps, 200))
    t0 = time.perf_counter()
    for i in range(e_steps):
        eng.decode_host(xhs[i % N_INPUTS].data_ptr(), T, oh.data_ptr())
    e2e_s = (time.perf_counter() - t0) / e_steps
    if dist:
        t = torch.tensor([e2e_s], device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = world * T / e2e_s
    eng.close()
    del eng

    # ---- n4 sweep (the metric's x axis) -------------------------------------
    sweep = []
    if args.sweep:
        for n4 in args.sweep_points:
            p, e = build(n4)
            e.synth_input(0, T)
            e.decode(T)
            e.sync()
            m = time_engine(moe, torch, e, T, max(20, min(args.steps, 100)), 3)
            fm, fb, _ = e.profile_step(T)
            sweep.append({"n4": n4, "tokens_per_s": round(T * 1000.0 / m, 2), "ms_per_step": round(m, 4),
                          "expert_gb_per_token": round(sum(fb) / 1e9 / T, 3),
                          "ffn_gbs": round(sum(fb) / (sum(fm) * 1e-3) / 1e9, 1)})
            e.close()
            del e

    # ---- decode batch sweep at the headline n4 (GEMV below tc_min, tcgen05 from there) ----
    batch = []
    if args.batch_sweep and args.batch_points:
        plan_b = moe.make_plan(moe.TaskRequest(moe.QUALITY, args.n4, 0), moe.HardwareProfile(10**15), prof)
        eng = moe.MoeEngine(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, plan_b, max_tokens=max(args.batch_points),
                            seed=args.seed + rank, device=device, norm_eps=NORM_EPS, tc_min_tokens=args.tc_min)
        for tb in args.batch_points:
            eng.synth_input(0, tb)
            eng.decode(tb)
            eng.sync()
            m = time_engine(moe, torch, eng, tb, max(5, min(args.steps, 30)), 3)
            batch.append({"batch": tb, "tokens_per_s": round(world * tb * 1000.0 / m, 1), "ms_per_step": round(m, 4),
                          "path": "tcgen05" if tb >= args.tc_min else "gemv"})
        eng.close()
        del eng

    # ---- prefill: one Mixtral layer, tcgen05 expert GEMM, TFLOP/s ----------
    prefill = []
    if args.prefill and args.prefill_points:
        prof1 = moe.profile_for_shape(D_MODEL, D_FFN, 1, EXPERTS, TOPK)
        tf_peak = _peak_tflops()
        for prec in (1, 0):
            plan1 = moe.assign_locations([prec] * EXPERTS, moe.HardwareProfile(10**15), prof1)
            eng = moe.MoeEngine(1, EXPERTS, TOPK, D_MODEL, D_FFN, plan1, max_tokens=max(args.prefill_points),
                                seed=args.seed + rank, device=device, norm_eps=NORM_EPS)
            for tp in args.prefill_points:
                eng.synth_input(1, tp)
                eng.decode(tp)
                eng.sync()
                fm = []
                for _ in range(4):
                    m_, _, _ = eng.profile_step(tp)
                    fm.append(m_[0])
                ffn = sorted(fm)[len(fm) // 2]
                flops = 6.0 * D_MODEL * D_FFN * tp * TOPK
                tf = flops / (ffn * 1e-3) / 1e12
                prefill.append({"tokens": tp, "experts": "bf16" if prec else "int4-g128", "ffn_ms": round(ffn, 4),
                                "tflops": round(tf, 1), "frac_of_peak": round(tf / tf_peak, 4)})
            eng.close()
            del eng

    # ---- C4: host-resident expert fraction streamed through the swap slot ----
    host_split = None
    if args.host_split and rank == 0:
        host_split = host_split_sweep(moe, torch, prof, args, device)

    # ---- f1: reconfiguration executor (plan -> plan on the device) ----
    reconfig = None
    if args.reconfig and rank == 0:
        reconfig = reconfig_sweep(moe, torch, args, device)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tps, cores, sample = cpu_port_tokens_per_s(plan.precision, T, seconds=args.cpu_seconds)
        cpu = {"value": round(tps, 4), "unit": "tokens/s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 / int4-g128 weights, bf16 activations, fp32 accumulate",
            "data": "synthetic (seeded counter-based generator, int4 = RTN-g128 of the bf16 masters)",
            "config": bench_config(args, T, world),
            "e2e": {"value": round(e2e, 3), "unit": "tokens/s", "h2d_bytes_per_step": T * D_MODEL * 2,
                    "d2h_bytes_per_step": T * D_MODEL * 2},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                         "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                         "traffic_note": traffic_note,
                         "kernel": kernel_desc,
                         "bytes_per_launch": round(avg_bytes), "ms_per_launch": round(avg_ms, 5),
                         "share_of_step": round(ffn_share, 4),
                         "frac_of_nominal_8000_gbs": round(achieved / 8000.0, 4)},
            "gpu_launches": kps * (args.steps),
            "kernels_per_step": kps,
            "clocks": clocks,
            "sweep": sweep,
            "batch_sweep": batch,
            "host_split": host_split,
            "reconfig": reconfig,
            "prefill_tcgen05": {"points": prefill, "peak_tflops": _peak_tflops(),
                                "peak_kind": "MEASURED_PEAKS bf16_tflops (burst)",
                                "flops": "6*d*f*T*k (gate/up + down, top-k=2)",
                                "timed": "expert FFN launches of one layer (gather, 2 x tcgen05 GEMM, combine)",
                                "kernels": "from 128 slots per expert: tc_ffn_wide2 (persistent, cta_group::2 "
                                           "M=256 x N=256 tiles, bf16 and int4 experts); below 128: "
                                           "tc_ffn_persist (128-token tiles, both passes in one launch)"},
            "cpu_baseline": cpu,
            "bytes_per_expert": {"bf16": s16, "int4_g128": s4},
        }
        print(json.dumps(line), flush=True)
        bad = [(r["resident_frac"], pol) for r in (host_split or {}).get("points", [])
               for pol in ("static", "lru") if pol in r and not r[pol]["counters_equal_simulate"]]
        if bad:  # the engine's counters must equal the reference cost model's on the exported routing
            print(f"counters_equal_simulate is false at {bad}", file=sys.stderr, flush=True)
            sys.exit(3)


def h2d_gbs(torch, device, nbytes=1 << 30):
    """Pinned host -> device copy bandwidth (cudaMemcpyAsync), best of 3."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    del src, dst
    return best


def host_split_sweep(moe, torch, prof, args, device):
    """C4: plan_quality(n4, budget) over budgets from full
    residency down to the non-expert + swap floor; host-resident experts live
    in a pinned arena and are re-streamed into the single swap slot on every
    activation (Static policy, simulator.cpp:98-106).  Reports measured
    tokens/s, the engine's counters == the reference cost model's simulate()
    on the exported routing, and expected_throughput with the measured H2D
    bandwidth and compute_penalty4 = 1."""
    bw = h2d_gbs(torch, device)
    n4 = args.host_split_n4
    s16, s4 = moe.expert_size(prof, 1), moe.expert_size(prof, 0)
    full = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), moe.HardwareProfile(10**15), prof)
    # model calibration: price the reference cost
    # model at the measured B200 costs -- per-activation compute from the
    # all-resident decode of this plan (CUDA events, graph replay), transfers
    # at the measured pinned H2D bandwidth, compute_penalty4 = 1
    eng = moe.MoeEngine(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, full, max_tokens=1, seed=args.seed, device=device,
                        norm_eps=NORM_EPS)
    eng.synth_input(0, 1)
    eng.decode(1)
    eng.sync()
    ms_res = time_engine(moe, torch, eng, 1, 40, 3)
    eng.close()
    del eng
    act_s = ms_res * 1e-3 / (LAYERS * TOPK)
    calib = moe.ModelProfile(**{**prof.__dict__, "compute_latency16_s": act_s, "compute_penalty4": 1.0,
                                "nonexpert_latency_s": 0.0})
    experts_bytes = sum(s4 if p == 0 else s16 for p in full.precision)
    floor = prof.size_nonexpert_bytes + max(s4 if n4 == LAYERS * EXPERTS else s16, s4)
    rows = []
    for frac in args.host_split_points:
        budget = int(floor + frac * experts_bytes)
        hw = moe.HardwareProfile(budget, bw * 1e9)
        try:
            plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), hw, prof)
        except moe.MoeError as exc:
            rows.append({"resident_frac": frac, "infeasible": str(exc)})
            continue
        model_tps = moe.expected_throughput(plan, calib, hw)
        row = {"resident_frac": frac, "gpu_budget_gb": round(budget / 1e9, 2), "experts_on_gpu": plan.n_gpu,
               "model_tps_expected_throughput": round(model_tps, 3)}
        # Static (the paper's scheme) and LRU (its Mixtral-Offloading baseline)
        for pol, cap in (("static", 0), ("lru", args.host_split_lru if plan.n_gpu < LAYERS * EXPERTS else 0)):
            if pol == "lru" and cap == 0:
                continue
            eng = moe.MoeEngine(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, plan, max_tokens=1, seed=args.seed,
                                device=device, norm_eps=NORM_EPS, use_graphs=True, lru_capacity=cap)
            eng.synth_input(0, 1)
            eng.decode(1)
            eng.sync()
            eng.reset_counters()
            trace = []
            steps = args.host_split_steps
            t0 = time.perf_counter()
            for st in range(steps):
                eng.synth_input(st + 1, 1)
                eng.decode(1)
                eng.sync()
                trace.extend(eng.last_routing(1))
            el = time.perf_counter() - t0
            c = eng.counters()
            sim = moe.simulate(plan, trace, steps, prof, hw, lru_capacity=cap)
            row[pol] = {"tokens_per_s": round(steps / el, 3), "hits": c.hits, "activations": c.activations,
                        "bytes_transferred": c.bytes_transferred, "lru_slots": cap,
                        "counters_equal_simulate": (c.activations, c.hits, c.bytes_transferred) ==
                                                   (sim.activations, sim.hits, sim.bytes_transferred)}
            eng.close()
            del eng
        rows.append(row)
    return {"n4": n4, "h2d_gbs_measured": round(bw, 1),
            "model_calibration": {"resident_ms_per_step": round(ms_res, 4), "compute_latency16_s": act_s,
                                  "compute_penalty4": 1.0, "nonexpert_latency_s": 0.0,
                                  "transfer_bw_bytes_per_s": bw * 1e9,
                                  "how": "all-resident decode of this plan (measured) / (layers x top_k); "
                                         "transfers at the measured pinned H2D bandwidth"},
            "policies": "static = single swap slot re-streamed per activation (planner.cpp:108, simulator.cpp:98-106); "
                        "lru = LRU cache of lru_slots device slots (simulator.cpp:37-62)",
            "steps_per_point": args.host_split_steps, "points": rows}


def reconfig_sweep(moe, torch, args, device):
    """MoeEngine.reconfigure between placement plans of a
    Mixtral-shaped stack of args.reconfig_layers layers (host copies of every
    expert in both precisions -- the reconfig model's CPU masters).  Per
    transition: the action list of diff_plans, the model's bytes_moved and
    est_downtime_s at the measured pinned H2D bandwidth, and the measured
    device time of the executed list; then one decode step checks the engine
    still runs."""
    L = args.reconfig_layers
    prof = moe.profile_for_shape(D_MODEL, D_FFN, L, EXPERTS, TOPK)
    s16, s4 = moe.expert_size(prof, 1), moe.expert_size(prof, 0)
    n = L * EXPERTS
    bw = h2d_gbs(torch, device) * 1e9
    full = n * s16 + 1
    steps = [("n4=0 resident", 0, full), ("n4=half, 1/2 of the experts' bytes", n // 2, n * (s16 + s4) // 4),
             ("n4=all resident", n, full), ("n4=0 resident", 0, full)]
    plans = [moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 7), moe.HardwareProfile(b, bw), prof) for _, n4, b in steps]
    eng = moe.MoeEngine(L, EXPERTS, TOPK, D_MODEL, D_FFN, plans[0], max_tokens=1, seed=args.seed, device=device,
                        norm_eps=NORM_EPS, keep_masters=True)
    rows = []
    # one untimed round first: the stream-ordered pool grows to the working set
    # (the engine keeps it mapped), so the reported round measures the moves
    for i in range(1, len(plans)):
        eng.reconfigure(plans[i], bw)
    for i in range(1, len(plans)):
        acts, _, _ = moe.diff_plans(plans[i - 1], plans[i], prof, moe.HardwareProfile(1, bw))
        kinds = {}
        for k, *_ in acts:
            name = ("offload", "fetch", "quantize", "dequantize")[k]
            kinds[name] = kinds.get(name, 0) + 1
        r = eng.reconfigure(plans[i], bw)
        eng.synth_input(0, 1)
        eng.decode(1)
        eng.sync()
        rows.append({"from": steps[i - 1][0], "to": steps[i][0], "experts_on_gpu": plans[i].n_gpu, "actions": kinds,
                     "bytes_moved": r["bytes_moved"], "bytes_h2d": r["bytes_h2d"],
                     "est_downtime_s": round(r["est_downtime_s"], 5), "measured_s": round(r["measured_s"], 5),
                     "measured_over_est": round(r["measured_s"] / r["est_downtime_s"], 3) if r["est_downtime_s"] else None})
    eng.close()
    return {"layers": L, "experts": n, "h2d_gbs_measured": round(bw / 1e9, 1), "round": "second (pool warm)",
            "model": "reconfig.cpp:57-82 (CPU->GPU bytes / transfer bw); Quantize of a resident expert runs the "
                     "int4-g128 quantiser on the device (not in the model's bytes)",
            "transitions": rows}


def _max_over_ranks(dist, v: float) -> float:
    import torch
    t = torch.tensor([v], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ep(args, rank, world, device):
    """Expert-parallel decode over `world` ranks: every rank's
    MoeEngine holds only its slots of each layer (slot s -> rank s*world//8)
    and T_local tokens (weak scaling); each layer sends only the routed token
    rows to their experts' owners and gets the outputs back over peer memory
    (ep_a2a.cu: NVLink P2P between GPUs, CUDA IPC handles), all inside the
    engine's graph-captured decode step.  torch.distributed (gloo) only
    carries the IPC handles, barriers and the max over ranks.  Timed with CUDA
    events on the engine stream between barriers, max over ranks.  Ranks may
    share a GPU (a 1-GPU box running --gpus 2): the exchange then crosses
    process contexts on one device -- correct, but time-sliced, so such a
    line measures the protocol, not NVLink."""
    import torch
    import torch.distributed as dist
    import paper_2407_14417_b200 as moe
    prof = moe.profile_for_shape(D_MODEL, D_FFN, LAYERS, EXPERTS, TOPK)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, args.n4, 0), moe.HardwareProfile(10**15), prof)
    T_local = args.tokens
    eng = moe.MoeEngine(LAYERS, EXPERTS, TOPK, D_MODEL, D_FFN, plan, max_tokens=T_local, seed=args.seed,
                        device=device, norm_eps=NORM_EPS, tc_min_tokens=args.tc_min, ep_rank=rank, ep_world=world)
    base, _ = eng.ep_buffer()
    handles = [None] * world
    dist.all_gather_object(handles, moe.ep_peer_ipc_handle(base))
    eng.ep_set_peers([base if r == rank else moe.ep_peer_ipc_open(handles[r]) for r in range(world)])
    shared_gpu = world > torch.cuda.device_count()
    n_in = 8
    for w in range(args.warmup):
        eng.synth_input(1000 + rank * n_in + (w % n_in), T_local)
        eng.decode(T_local)
    eng.sync()
    dist.barrier()
    steps = max(5, min(args.steps, 10 if shared_gpu else 100))
    stream = torch.cuda.ExternalStream(eng.stream_ptr)
    ms_total = 0.0
    with ClockSampler(device) as clk:
        per = max(1, steps // n_in)
        done = 0
        for i in range(n_in):
            k = per if i < n_in - 1 else steps - done
            if k <= 0:
                break
            eng.synth_input(1000 + rank * n_in + i, T_local)
            eng.decode(T_local)  # this input's first step, untimed
            eng.sync()
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(stream)
            for _ in range(k):
                eng.decode(T_local)
            end.record(stream)
            end.synchronize()
            ms_total += start.elapsed_time(end)
            done += k
    clocks = clk.summary()
    ms = _max_over_ranks(dist, ms_total / done)
    # per-rank algorithmic bytes of the last step: the distinct experts of this
    # rank's slots selected by any rank's tokens, per layer
    routes = [None] * world
    dist.all_gather_object(routes, eng.last_routing(T_local))
    sel = [set() for _ in range(LAYERS)]
    for r in range(world):
        for t in range(T_local):
            for l in range(LAYERS):
                for j in range(TOPK):
                    sel[l].add(routes[r][(t * LAYERS + l) * TOPK + j])
    b16, b4 = moe.expert_size(prof, moe.MOE_P16), moe.expert_size(prof, moe.MOE_P4)
    prec = plan.precision
    mine = [s for s in range(EXPERTS) if s * world // EXPERTS == rank]
    my_bytes = sum((b16 if prec[l * EXPERTS + s] == moe.MOE_P16 else b4) for l in range(LAYERS) for s in sel[l]
                   if s in mine)
    max_bytes = _max_over_ranks(dist, float(my_bytes))
    # e2e through the public API: pinned host tokens in, output back, every step
    xh = torch.empty(T_local * D_MODEL, dtype=torch.int16).pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    eng.synth_input(1000 + rank * n_in, T_local)
    eng.sync()
    xh.copy_(torch.as_tensor(_DevBytes(eng.input_ptr, T_local * D_MODEL * 2), device=f"cuda:{device}").view(torch.int16).cpu())
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        eng.decode_host(xh.data_ptr(), T_local, oh.data_ptr())
    e2e_s = _max_over_ranks(dist, (time.perf_counter() - t0) / steps)
    mem = eng.memory()
    expert_gb = _max_over_ranks(dist, mem["expert_bytes"] / 1e9)
    eng.close()
    if rank == 0:
        peak, peak_kind = peaks()
        achieved = max_bytes / (ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": round(world * T_local * 1000.0 / ms, 3), "unit": "tokens/s", "n_gpus": world,
            "steps": done, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16 / int4-g128 weights, bf16 activations, fp32 accumulate",
            "data": "synthetic (seeded counter-based generator)",
            "config": {"workload": "mixtral8x7b-shape 32-layer MoE stack, expert-parallel batch-%d/GPU decode" % T_local,
                       "n4": args.n4, "of": LAYERS * EXPERTS, "layer": "x + MoE(RMSNorm(x))",
                       "parallelism": "ep%d" % world, "experts_per_gpu_per_layer": len(mine),
                       "expert_gb_per_gpu": round(expert_gb, 3),
                       "exchange": "routed-row all-to-all over peer memory inside the engine step (ep_a2a.cu): "
                                   "dispatch 2*d B per routed (token, expert), return 4*d B",
                       "exchange_bytes_per_layer_per_gpu": {"dispatch": T_local * TOPK * D_MODEL * 2,
                                                            "return": T_local * TOPK * D_MODEL * 4},
                       "ranks_share_gpu": shared_gpu, "batch_per_gpu": T_local,
                       "inputs": "8 distinct synthetic token inputs per rank",
                       "l2": "no flush: every step streams GBs of distinct expert weights per GPU"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "what": "busiest rank's selected-expert bytes per step / step time (exchange and routing "
                                 "included in the time)"},
            "e2e": {"value": round(world * T_local / e2e_s, 3), "unit": "tokens/s",
                    "h2d_bytes_per_step": world * T_local * D_MODEL * 2, "d2h_bytes_per_step": world * T_local * D_MODEL * 2,
                    "how": "moe_engine_decode_host per rank (pinned H2D, step, D2H, sync), max over ranks"},
            # per layer: route, dispatch, wait, keys, permute, (gather), FFN (permute_rows, 2 streams, 2 finalizes
            # or gather + 2 tcgen05 + ...), return, wait, combine; + 1 epoch bump per step
            "gpu_launches": (13 * LAYERS + 1) * done, "clocks": clocks, "cpu_baseline": None,
            "note": "expert parallel (not replicas): every GPU holds and computes only its slots of each layer",
        }
        print(json.dumps(line), flush=True)


class _DevBytes:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n4", type=int, default=128)
    ap.add_argument("--tokens", type=int, default=1, help="decode batch T")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-sweep", dest="sweep", action="store_false")
    ap.add_argument("--sweep-points", type=lambda s: [int(v) for v in s.split(",")],
                    default=[0, 32, 64, 96, 128, 160, 192, 224, 256])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of expert parallel")
    ap.add_argument("--no-batch-sweep", dest="batch_sweep", action="store_false")
    ap.add_argument("--tc-min", type=int, default=32, help="batch-sweep engine: tcgen05 expert GEMM from this T")
    ap.add_argument("--batch-points", type=lambda s: [int(v) for v in s.split(",")] if s else [],
                    default=[1, 8, 32, 64, 128, 256])
    ap.add_argument("--no-prefill", dest="prefill", action="store_false")
    ap.add_argument("--no-host-split", dest="host_split", action="store_false")
    ap.add_argument("--host-split-n4", type=int, default=256)
    ap.add_argument("--host-split-points", type=lambda s: [float(v) for v in s.split(",")] if s else [],
                    default=[1.0, 0.75, 0.5, 0.25, 0.0])
    ap.add_argument("--host-split-steps", type=int, default=8)
    ap.add_argument("--host-split-lru", type=int, default=16, help="LRU device slots for the host-split LRU column")
    ap.add_argument("--no-reconfig", dest="reconfig", action="store_false")
    ap.add_argument("--reconfig-layers", type=int, default=4, help="Mixtral-shaped layers of the reconfig stack")
    ap.add_argument("--prefill-points", type=lambda s: [int(v) for v in s.split(",")] if s else [],
                    default=[512, 2048, 4096])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--shape", choices=["mixtral", "tiny"], default="mixtral",
                    help="tiny = BASELINE configs[0] (2 layers, d=512, ffn=1792) for quick checks; the bench "
                         "line is always the Mixtral shape")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.shape == "tiny":
        global D_MODEL, D_FFN, LAYERS
        D_MODEL, D_FFN, LAYERS = 512, 1792, 2

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: relaunch this command under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"--gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    ndev = max(1, torch.cuda.device_count())
    local = local % ndev  # more ranks than GPUs (a 1-GPU box running --gpus 2): ranks share devices
    torch.cuda.set_device(local)
    ep_mode = world > 1 and not args.replicas
    if world > 1:
        import torch.distributed as dist
        # the expert-parallel exchange is the engine's own (peer memory); the
        # process group only carries handles / barriers / maxima -> gloo, which
        # also works when ranks share a GPU (NCCL refuses duplicate devices)
        if ep_mode or world > ndev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if ep_mode:
        run_ep(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
