"""MoeEngine parity: the B200 MoE-layer forward vs the CPU oracle, and its
SimReport counters vs the reference simulate() on the exported routing.

Config C1 of BASELINE.json (tiny: 2 layers, 8 experts top-2, d=512,
ffn=1792, 4 of 8 experts per layer int4 via assign_quantization(8, seed=1),
32-token decode) and C2 (one Mixtral-shaped layer, all-bf16 vs all-int4).
"""
import numpy as np
import pytest

from helpers import MIXTRAL, RTOL_BF16, TINY, assert_close, assert_delta_close, bf16_to_f32, read_device, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod(cuda):
    import torch
    return torch


def quality_plan(moe, cfg, n4, seed, budget=10**15):
    prof = moe.profile_for_shape(cfg["d_model"], cfg["d_ffn"], cfg["num_layers"], cfg["experts_per_layer"],
                                 cfg["top_k"])
    return prof, moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, seed), moe.HardwareProfile(budget), prof)


def make_engine(moe, cfg, plan, seed, T=1, graphs=True, eps=0.0, tc_min=0):
    return moe.MoeEngine(cfg["num_layers"], cfg["experts_per_layer"], cfg["top_k"], cfg["d_model"], cfg["d_ffn"],
                         plan, max_tokens=T, seed=seed, use_graphs=graphs, norm_eps=eps, tc_min_tokens=tc_min)


def layer_precisions(plan, layer, E):
    return plan.precision[layer * E:(layer + 1) * E]


def test_tiny_plan_is_4_of_8_per_layer(moe):
    _, plan = quality_plan(moe, TINY, 8, 1)
    assert [sum(1 for p in plan.precision[l * 8:(l + 1) * 8] if p == 0) for l in range(2)] == [4, 4]
    assert plan.n_gpu == 16


@pytest.mark.parametrize("eps", [0.0, 1e-5])
@pytest.mark.parametrize("T", [1, 3, 4, 8])
def test_tiny_layer_parity(moe, orc, torch_mod, cuda, T, eps):
    """eps > 0: the decoder-layer RMSNorm fused into the route kernel --
    normalised x must be bit-identical to the oracle's (logits are)."""
    torch = torch_mod
    seed = 42
    _, plan = quality_plan(moe, TINY, 8, 1)
    eng = make_engine(moe, TINY, plan, seed, T, eps=eps)
    m = orc.model(2, 8, 2, 512, 1792, seed, eps)
    x = orc.step_input(m, 0, T)
    for layer in range(2):
        prec = layer_precisions(plan, layer, 8)
        out_ref, idx_ref, w_ref, lg_ref = orc.moe_layer(m, layer, prec, x, T)
        xd = to_dev(x, torch, cuda)
        out = torch.empty(T * 512, dtype=torch.int16, device=cuda)
        idx = torch.empty(T * 2, dtype=torch.int32, device=cuda)
        w = torch.empty(T * 2, dtype=torch.float32, device=cuda)
        lg = torch.empty(T * 8, dtype=torch.float32, device=cuda)
        eng.forward_layer(layer, xd, T, out, idx, w, lg)
        eng.sync()
        assert np.array_equal(to_np(lg, np.float32).view(np.uint32).reshape(T, 8), lg_ref.view(np.uint32))
        assert np.array_equal(to_np(idx, np.int32).reshape(T, 2), idx_ref)
        got = to_np(out, np.uint16).reshape(T, 512)
        assert_close(bf16_to_f32(got), bf16_to_f32(out_ref), RTOL_BF16, f"layer {layer}")
        assert_delta_close(got, out_ref, x, what=f"layer {layer}")
        x = got  # feed the GPU's output to the next layer (per-layer parity on identical inputs)
    eng.close()


@pytest.mark.parametrize("eps", [0.0, 1e-5])
def test_tiny_decode_32_steps(moe, orc, torch_mod, cuda, eps):
    """C1: 32-token decode through the stack (CUDA graph), vs the oracle
    stack run free on the same step inputs."""
    torch = torch_mod
    seed = 42
    prof, plan = quality_plan(moe, TINY, 8, 1)
    eng = make_engine(moe, TINY, plan, seed, 1, graphs=True, eps=eps)
    m = orc.model(2, 8, 2, 512, 1792, seed, eps)
    flips = 0
    for step in range(32):
        eng.synth_input(step, 1)
        eng.decode(1)
        got = read_device(torch, eng.output_ptr, 512 * 2).view(np.uint16)
        x = orc.step_input(m, step, 1)
        routing = []
        for layer in range(2):
            x, idx_ref, _, _ = orc.moe_layer(m, layer, layer_precisions(plan, layer, 8), x, 1)
            routing.extend(sorted(idx_ref[0].tolist()))
        assert_close(bf16_to_f32(got), bf16_to_f32(x), RTOL_BF16, f"step {step}")
        flips += routing != eng.last_routing(1)
    assert flips == 0
    c = eng.counters()
    assert c.tokens == 32 and c.activations == 32 * 2 * 2 and c.hits == c.activations
    eng.close()


def test_graph_equals_eager(moe, orc, torch_mod, cuda):
    torch = torch_mod
    _, plan = quality_plan(moe, TINY, 8, 1)
    outs = []
    for graphs in (True, False):
        eng = make_engine(moe, TINY, plan, 7, 4, graphs=graphs)
        eng.synth_input(3, 4)
        eng.decode(4)
        eng.sync()
        outs.append(read_device(torch, eng.output_ptr, 4 * 512 * 2))
        eng.close()
    assert np.array_equal(outs[0], outs[1])


def test_decode_host_equals_device(moe, torch_mod, cuda):
    torch = torch_mod
    _, plan = quality_plan(moe, TINY, 8, 1)
    eng = make_engine(moe, TINY, plan, 9, 2)
    eng.synth_input(5, 2)
    eng.decode(2)
    eng.sync()
    dev_out = read_device(torch, eng.output_ptr, 2 * 512 * 2)
    x = read_device(torch, eng.input_ptr, 2 * 512 * 2)
    out = np.empty_like(x)
    eng.decode_host(x.ctypes.data, 2, out.ctypes.data)
    assert np.array_equal(out, dev_out)
    eng.close()


@pytest.mark.parametrize("budget_frac", [0.5, 0.25, 0.0])
def test_host_streaming_counters_match_simulate(moe, ref, torch_mod, cuda, budget_frac):
    """C4 semantics on the tiny shape: host-resident experts streamed into the
    swap slot (Static).  Counters == reference simulate() on the exported
    routing; outputs identical to the all-resident engine."""
    torch = torch_mod
    prof = moe.profile_for_shape(512, 1792, 2)
    n4 = 8
    full = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 1), moe.HardwareProfile(10**15), prof)
    foot = moe.gpu_footprint(full, prof)
    s16 = moe.expert_size(prof, 1)
    budget = int(prof.size_nonexpert_bytes + s16 + budget_frac * (foot - prof.size_nonexpert_bytes))
    hw = moe.HardwareProfile(budget)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 1), hw, prof)
    assert plan.n_gpu < 16
    st, rprec, rloc, rswap = ref.make_plan(prof, budget, hw.transfer_bw_bytes_per_s, 1, n4, 1)
    assert st == 0 and list(rprec) == plan.precision and list(rloc) == plan.location and rswap == plan.swap_slot_bytes

    eng = make_engine(moe, TINY, plan, 11, 1)
    base = make_engine(moe, TINY, full, 11, 1)
    trace = []
    for step in range(12):
        for e in (eng, base):
            e.synth_input(step, 1)
            e.decode(1)
            e.sync()
        a = read_device(torch, eng.output_ptr, 1024)
        b = read_device(torch, base.output_ptr, 1024)
        assert np.array_equal(a, b), "streamed experts must compute bit-identically"
        trace.extend(eng.last_routing(1))
    c = eng.counters()
    st, sim = ref.simulate(prof, hw.transfer_bw_bytes_per_s, plan.precision, plan.location, plan.swap_slot_bytes,
                           12, np.array(trace, np.int32))
    assert st == 0
    assert (c.activations, c.hits, c.bytes_transferred) == (sim[0], sim[1], sim[2])
    mine = moe.simulate(plan, trace, 12, prof, hw)
    assert (mine.activations, mine.hits, mine.bytes_transferred) == (sim[0], sim[1], sim[2])
    # f4: the engine's real routing as a v1 trace file the reference tools replay
    doc = moe.write_trace(prof, 12, trace)
    assert doc == ref.write_trace(prof, 12, np.array(trace, np.int32))
    tr = moe.read_trace(doc)
    assert tr["slots"] == trace and tr["fingerprint"] == moe.profile_fingerprint(prof)
    assert moe.read_plan(moe.write_plan(plan, prof), prof) == plan
    eng.close()
    base.close()


@pytest.mark.parametrize("precision", [1, 0])
@pytest.mark.parametrize("T", [1, 4])
def test_mixtral_layer_parity(moe, orc, torch_mod, cuda, precision, T):
    """C2: one Mixtral-shaped layer (d=4096, f=14336, 8 experts top-2), all-bf16
    vs all-int4, on identical inputs."""
    torch = torch_mod
    cfg = dict(MIXTRAL, num_layers=1)
    prof = moe.profile_for_shape(4096, 14336, 1)
    plan = moe.assign_locations([precision] * 8, moe.HardwareProfile(10**15), prof)
    eng = make_engine(moe, cfg, plan, 2024, T)
    m = orc.model(1, 8, 2, 4096, 14336, 2024)
    x = orc.step_input(m, 0, T)
    out_ref, idx_ref, _, lg_ref = orc.moe_layer(m, 0, [precision] * 8, x, T)
    out = torch.empty(T * 4096, dtype=torch.int16, device=cuda)
    idx = torch.empty(T * 2, dtype=torch.int32, device=cuda)
    w = torch.empty(T * 2, dtype=torch.float32, device=cuda)
    lg = torch.empty(T * 8, dtype=torch.float32, device=cuda)
    eng.forward_layer(0, to_dev(x, torch, cuda), T, out, idx, w, lg)
    eng.sync()
    assert np.array_equal(to_np(lg, np.float32).view(np.uint32).reshape(T, 8), lg_ref.view(np.uint32))
    assert np.array_equal(to_np(idx, np.int32).reshape(T, 2), idx_ref)
    assert_close(bf16_to_f32(to_np(out, np.uint16).reshape(T, 4096)), bf16_to_f32(out_ref), RTOL_BF16,
                 f"mixtral layer {'bf16' if precision else 'int4'}")
    assert_delta_close(to_np(out, np.uint16).reshape(T, 4096), out_ref, x, what="mixtral layer")
    eng.close()


def test_mixtral_stack_prenorm_is_finite(moe, torch_mod, cuda):
    """C3 workload sanity: the full 32-layer Mixtral-shaped stack with the
    decoder-layer RMSNorm stays finite and routes k distinct experts in every
    layer (without the norm the synthetic residual stream overflows and the
    routing degenerates -- a bench on it would be invalid)."""
    torch = torch_mod
    cfg = dict(MIXTRAL)
    prof = moe.profile_for_shape(4096, 14336, 32)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 128, 0), moe.HardwareProfile(10**15), prof)
    eng = make_engine(moe, cfg, plan, 0, 1, graphs=True, eps=1e-5)
    for step in range(4):
        eng.synth_input(step, 1)
        eng.decode(1)
        eng.sync()
        out = bf16_to_f32(read_device(torch, eng.output_ptr, 4096 * 2).view(np.uint16))
        assert np.isfinite(out).all()
        r = eng.last_routing(1)
        assert all(r[2 * l] != r[2 * l + 1] for l in range(32))
    eng.close()


@pytest.mark.parametrize("eps", [0.0, 1e-5])
@pytest.mark.parametrize("T", [32, 100, 520])
def test_tiny_layer_parity_tcgen05(moe, orc, torch_mod, cuda, T, eps):
    """Batched decode through the engine's tcgen05 expert GEMM (T >= tc_min):
    routing bit-exact, layer output within tolerance, mixed int4/bf16 plan."""
    torch = torch_mod
    seed = 17
    _, plan = quality_plan(moe, TINY, 8, 1)
    eng = make_engine(moe, TINY, plan, seed, T, eps=eps, tc_min=16)
    m = orc.model(2, 8, 2, 512, 1792, seed, eps)
    x = orc.step_input(m, 3, T)
    for layer in range(2):
        out_ref, idx_ref, _, lg_ref = orc.moe_layer(m, layer, layer_precisions(plan, layer, 8), x, T)
        out = torch.empty(T * 512, dtype=torch.int16, device=cuda)
        idx = torch.empty(T * 2, dtype=torch.int32, device=cuda)
        w = torch.empty(T * 2, dtype=torch.float32, device=cuda)
        lg = torch.empty(T * 8, dtype=torch.float32, device=cuda)
        eng.forward_layer(layer, to_dev(x, torch, cuda), T, out, idx, w, lg)
        eng.sync()
        assert np.array_equal(to_np(lg, np.float32).view(np.uint32).reshape(T, 8), lg_ref.view(np.uint32))
        assert np.array_equal(to_np(idx, np.int32).reshape(T, 2), idx_ref)
        got = to_np(out, np.uint16).reshape(T, 512)
        assert_close(bf16_to_f32(got), bf16_to_f32(out_ref), RTOL_BF16, f"layer {layer}")
        assert_delta_close(got, out_ref, x, what=f"layer {layer} tcgen05")
        x = got
    eng.close()


@pytest.mark.parametrize("precision", [1, 0])
def test_mixtral_layer_parity_tcgen05(moe, orc, torch_mod, cuda, precision):
    """C5-shaped batch (128 tokens) on one Mixtral layer through tcgen05."""
    torch = torch_mod
    T = 128
    cfg = dict(MIXTRAL, num_layers=1)
    prof = moe.profile_for_shape(4096, 14336, 1)
    plan = moe.assign_locations([precision] * 8, moe.HardwareProfile(10**15), prof)
    eng = make_engine(moe, cfg, plan, 2025, T, eps=1e-5)
    m = orc.model(1, 8, 2, 4096, 14336, 2025, 1e-5)
    x = orc.step_input(m, 0, T)
    out_ref, idx_ref, _, _ = orc.moe_layer(m, 0, [precision] * 8, x, T)
    out = torch.empty(T * 4096, dtype=torch.int16, device=cuda)
    idx = torch.empty(T * 2, dtype=torch.int32, device=cuda)
    eng.forward_layer(0, to_dev(x, torch, cuda), T, out, idx)
    eng.sync()
    assert np.array_equal(to_np(idx, np.int32).reshape(T, 2), idx_ref)
    assert_close(bf16_to_f32(to_np(out, np.uint16).reshape(T, 4096)), bf16_to_f32(out_ref), RTOL_BF16,
                 f"mixtral layer tcgen05 {'bf16' if precision else 'int4'}")
    eng.close()


@pytest.mark.parametrize("cap", [2, 4, 7])
def test_lru_counters_match_simulate(moe, ref, torch_mod, cuda, cap):
    """§8f row f2: LRU residency (simulator.cpp:37-62) -- host-resident
    experts cached in `cap` device slots.  hits / bytes_transferred equal the
    reference simulate(Lru, cap) on the exported routing; outputs stay
    bit-identical to the all-resident engine."""
    torch = torch_mod
    prof = moe.profile_for_shape(512, 1792, 2)
    full = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    s16 = moe.expert_size(prof, 1)
    budget = int(prof.size_nonexpert_bytes + s16 + 0.3 * (moe.gpu_footprint(full, prof) - prof.size_nonexpert_bytes))
    hw = moe.HardwareProfile(budget)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), hw, prof)
    assert plan.n_gpu < 16
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plan, max_tokens=1, seed=11, lru_capacity=cap)
    base = make_engine(moe, TINY, full, 11, 1)
    trace = []
    steps = 16
    for step in range(steps):
        for e in (eng, base):
            e.synth_input(step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, eng.output_ptr, 1024), read_device(torch, base.output_ptr, 1024))
        trace.extend(eng.last_routing(1))
    c = eng.counters()
    st, sim = ref.simulate(prof, hw.transfer_bw_bytes_per_s, plan.precision, plan.location, plan.swap_slot_bytes,
                           steps, np.array(trace, np.int32), cap)
    assert st == 0
    assert (c.activations, c.hits, c.bytes_transferred) == (sim[0], sim[1], sim[2])
    static = moe.simulate(plan, trace, steps, prof, hw)
    assert c.hits >= static.hits  # caching never loses hits
    eng.close()
    base.close()


def test_measured_pareto_sweep_tiny(moe, cuda):
    """f3: measured columns next to the simulated ones (tiny shape).  Fully
    resident cells hit every activation."""
    from paper_2407_14417_b200 import pareto
    shape = (2, 8, 2, 512, 1792)
    prof = moe.profile_for_shape(512, 1792, 2)
    s16 = moe.expert_size(prof, 1)
    budgets = [prof.size_nonexpert_bytes + 4 * s16, prof.size_nonexpert_bytes + 16 * s16]
    rows, meas = pareto.measured_sweep(moe, budgets, [0, 16], shape, 12.285e9, 20, seed=3, steps=6)
    assert len(rows) == 4
    for r, m in zip(rows, meas):
        assert r.feasible and m is not None and m[0] > 0
        if r.n_gpu == 16:
            assert r.report.hit_rate == 1.0 and m[1] == 1.0
        else:
            assert 0.0 <= m[1] <= 1.0
    doc = moe.pareto_csv(rows, meas)
    assert len(doc.splitlines()) == 5 and ",-,-" not in doc


@pytest.mark.parametrize("graphs", [True, False])
def test_reconfigure_executor_bit_identical(moe, torch_mod, cuda, graphs):
    """f1: reconfigure A -> B -> C on the device; every decode after a
    reconfiguration is bit-identical to a fresh engine built with that plan,
    the measured H2D bytes equal the model's bytes_moved, and the counters
    equal simulate() on the new plan."""
    torch = torch_mod
    prof = moe.profile_for_shape(512, 1792, 2)
    s16, s4 = moe.expert_size(prof, 1), moe.expert_size(prof, 0)
    full = 16 * s16 + 1
    plans = [moe.make_plan(moe.TaskRequest(moe.QUALITY, 4, 1), moe.HardwareProfile(full), prof),
             moe.make_plan(moe.TaskRequest(moe.QUALITY, 12, 2), moe.HardwareProfile(4 * s16 + 2 * s4 + 1), prof),
             moe.make_plan(moe.TaskRequest(moe.QUALITY, 2, 3), moe.HardwareProfile(9 * s16 + 1), prof),
             moe.make_plan(moe.TaskRequest(moe.QUALITY, 4, 1), moe.HardwareProfile(full), prof)]
    kinds = set()
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plans[0], max_tokens=2, seed=21, use_graphs=graphs, norm_eps=1e-5,
                        keep_masters=True)
    for i, target in enumerate(plans[1:], 1):
        acts, nbytes, _ = moe.diff_plans(plans[i - 1], target, prof, moe.HardwareProfile(1))
        kinds |= {a[0] for a in acts}
        rep = eng.reconfigure(target, 50e9)
        assert rep["actions"] == len(acts) and rep["bytes_moved"] == nbytes and rep["bytes_h2d"] == nbytes
        fresh = moe.MoeEngine(2, 8, 2, 512, 1792, target, max_tokens=2, seed=21, use_graphs=graphs, norm_eps=1e-5)
        eng.reset_counters()
        trace = []
        for step in range(6):
            for e in (eng, fresh):
                e.synth_input(step, 2)
                e.decode(2)
                e.sync()
            assert np.array_equal(read_device(torch, eng.output_ptr, 2 * 512), read_device(torch, fresh.output_ptr, 2 * 512))
            trace.extend(eng.last_routing(2))
        c = eng.counters()
        sim = moe.simulate(target, trace, 12, prof, moe.HardwareProfile(1))
        assert (c.activations, c.hits, c.bytes_transferred) == (sim.activations, sim.hits, sim.bytes_transferred)
        fresh.close()
    assert kinds == {moe.OFFLOAD, moe.FETCH, moe.QUANTIZE, moe.DEQUANTIZE}
    eng.close()


def test_reconfigure_needs_masters(moe, cuda):
    prof = moe.profile_for_shape(512, 1792, 2)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 4, 1), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plan, seed=1)
    with pytest.raises(moe.UsageError):
        eng.reconfigure(plan, 50e9)
    eng.close()


def test_reconfigure_with_lru_cache(moe, torch_mod, cuda):
    """f1 x f2: an LRU engine reconfigured to a plan with a different host set
    starts from an empty cache; its counters equal simulate(Lru) on the new
    plan and its outputs equal a fresh all-resident engine."""
    torch = torch_mod
    prof = moe.profile_for_shape(512, 1792, 2)
    s16 = moe.expert_size(prof, 1)
    full = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    a = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(6 * s16), prof)
    b = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(4 * s16), prof)
    assert a.location != b.location and b.n_gpu < 16
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, a, max_tokens=1, seed=11, lru_capacity=3, keep_masters=True)
    base = make_engine(moe, TINY, full, 11, 1)
    for step in range(4):
        eng.synth_input(step, 1)
        eng.decode(1)
    eng.sync()
    eng.reconfigure(b, 50e9)
    eng.reset_counters()
    trace = []
    for step in range(10):
        for e in (eng, base):
            e.synth_input(step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, eng.output_ptr, 1024), read_device(torch, base.output_ptr, 1024))
        trace.extend(eng.last_routing(1))
    c = eng.counters()
    sim = moe.simulate(b, trace, 10, prof, moe.HardwareProfile(1), lru_capacity=3)
    assert (c.activations, c.hits, c.bytes_transferred) == (sim.activations, sim.hits, sim.bytes_transferred)
    eng.close()
    base.close()


def _host_plan(moe, frac, n4=8, seed=1):
    prof = moe.profile_for_shape(512, 1792, 2)
    full = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, seed), moe.HardwareProfile(10**15), prof)
    s16 = moe.expert_size(prof, 1)
    budget = int(prof.size_nonexpert_bytes + s16 + frac * (moe.gpu_footprint(full, prof) - prof.size_nonexpert_bytes))
    hw = moe.HardwareProfile(budget)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, seed), hw, prof)
    assert plan.n_gpu < 16
    return prof, full, plan, hw


@pytest.mark.parametrize("cap,T", [(2, 2), (2, 4), (3, 4), (5, 8)])
def test_lru_batched_outputs_match_resident(moe, torch_mod, cuda, cap, T):
    """with T > 1 an expert that hit in the LRU cache can be
    evicted by a later activation of the same layer before it is computed.
    The engine computes every host expert at its first activation, from the
    slot it holds then, so outputs stay bit-identical to the all-resident
    engine for T * k > capacity."""
    torch = torch_mod
    prof, full, plan, hw = _host_plan(moe, 0.3)
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plan, max_tokens=T, seed=11, lru_capacity=cap)
    base = make_engine(moe, TINY, full, 11, T)
    static = moe.MoeEngine(2, 8, 2, 512, 1792, plan, max_tokens=T, seed=11)
    trace = []
    for step in range(10):
        for e in (eng, base, static):
            e.synth_input(step, T)
            e.decode(T)
            e.sync()
        want = read_device(torch, base.output_ptr, T * 1024)
        assert np.array_equal(read_device(torch, eng.output_ptr, T * 1024), want), f"LRU step {step}"
        assert np.array_equal(read_device(torch, static.output_ptr, T * 1024), want), f"Static step {step}"
        trace.extend(eng.last_routing(T))
    # Static counters equal simulate() at any batch size (no order dependence)
    c = static.counters()
    sim = moe.simulate(plan, trace, 10 * T, prof, hw)
    assert (c.activations, c.hits, c.bytes_transferred) == (sim.activations, sim.hits, sim.bytes_transferred)
    cl = eng.counters()
    assert cl.activations == c.activations and cl.hits >= c.hits
    for e in (eng, base, static):
        e.close()


@pytest.mark.parametrize("cap", [0, 3])
def test_counters_after_warmup_reset_match_simulate(moe, torch_mod, cuda, cap):
    """The bench's host-split protocol: a warm-up decode, reset_counters(),
    then N timed steps.  reset_counters() opens a new simulate() window (the
    LRU accounting cache starts cold, as simulate() does), so the counters
    equal simulate() on the post-reset trace (LRU mismatch)."""
    prof, full, plan, hw = _host_plan(moe, 0.3)
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plan, max_tokens=1, seed=11, lru_capacity=cap)
    for step in range(3):
        eng.synth_input(100 + step, 1)
        eng.decode(1)
    eng.sync()
    eng.reset_counters()
    trace = []
    for step in range(12):
        eng.synth_input(step, 1)
        eng.decode(1)
        eng.sync()
        trace.extend(eng.last_routing(1))
    c = eng.counters()
    sim = moe.simulate(plan, trace, 12, prof, hw, lru_capacity=cap)
    assert (c.activations, c.hits, c.bytes_transferred) == (sim.activations, sim.hits, sim.bytes_transferred)
    eng.close()


@pytest.mark.parametrize("lru", [0, 4])
def test_host_split_tcgen05_batch(moe, torch_mod, cuda, lru):
    """Batched decode (T >= tc_min_tokens, tcgen05) with host-resident
    experts streamed through the swap slot(s): bit-identical to the
    all-resident engine on the same path."""
    torch = torch_mod
    T = 40
    prof, full, plan, hw = _host_plan(moe, 0.4)
    eng = moe.MoeEngine(2, 8, 2, 512, 1792, plan, max_tokens=T, seed=5, tc_min_tokens=16, lru_capacity=lru,
                        norm_eps=1e-5)
    base = moe.MoeEngine(2, 8, 2, 512, 1792, full, max_tokens=T, seed=5, tc_min_tokens=16, norm_eps=1e-5)
    for step in range(3):
        for e in (eng, base):
            e.synth_input(step, T)
            e.decode(T)
            e.sync()
        assert np.array_equal(read_device(torch, eng.output_ptr, T * 1024), read_device(torch, base.output_ptr, T * 1024))
    c = eng.counters()
    assert c.activations == 3 * T * 2 * 2 and c.bytes_transferred > 0
    eng.close()
    base.close()


_COMBINE_PROBE = r"""
import hashlib, os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2407_14417_b200 as moe
from helpers import read_device
prof = moe.profile_for_shape(4096, 14336, 2, 8, 2)
plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 3), moe.HardwareProfile(10**15), prof)
eng = moe.MoeEngine(2, 8, 2, 4096, 14336, plan, max_tokens=64, seed=9, norm_eps=1e-5, tc_min_tokens=32)
h = hashlib.sha256()
for step in range(3):
    eng.synth_input(40 + step, 64)
    eng.decode(64)
    eng.sync()
    h.update(read_device(torch, eng.output_ptr, 64 * 4096 * 2).tobytes())
print(h.hexdigest())
"""


def test_tc_combine_from_split_partials_bitexact(moe, cuda):
    """moek_ffn_tc_combine: the K5 combine read straight from the fused launch's
    down-pass split partials gives the same bits as split_reduce + combine
    (MOE_TC_DBG bit 22), on a mixed bf16/int4 Mixtral-shaped stack at T = 64."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    digests = []
    for dbg in ("0", "4194304"):
        env = dict(os.environ, MOE_TC_DBG=dbg)
        r = subprocess.run([sys.executable, "-c", _COMBINE_PROBE], cwd=root, env=env, capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        digests.append(r.stdout.strip().splitlines()[-1])
    assert digests[0] == digests[1]
