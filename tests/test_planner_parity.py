"""The placement config and control-plane host API (C ABI) vs the reference.

Known-answer tests restate the reference's own doctest suites
(tests/test_planner.cpp, tests/test_profiles.cpp) against our C++
re-implementation through the C ABI; the `ref`-fixture tests compare
bit-for-bit with the reference library compiled from /root/reference
(oracle/_ref) on seeded random cases, mirroring the reference's property
suites (test_planner.cpp:235-320) at their case counts.
"""
import numpy as np
import pytest

MIX_BW = 336_000_000.0 / 0.02735


@pytest.fixture(scope="module")
def kM(moe):
    return moe.mixtral_sec41()


def hw(moe, budget):
    return moe.HardwareProfile(budget, MIX_BW)


def toy(moe):
    # test_planner.cpp:37-48
    return moe.ModelProfile(num_layers=2, experts_per_layer=2, top_k=1, size_nonexpert_bytes=1000,
                            size_expert16_bytes=400, quant_ratio=4.0, compute_latency16_s=0.0, nonexpert_latency_s=0.0)


# ----------------------------------------------------------- test_profiles.cpp
def test_empty_document_defaults(moe):
    m, h = moe.load_profiles("")
    assert (m.num_layers, m.experts_per_layer, m.num_experts, m.top_k) == (32, 8, 256, 2)
    assert (m.size_nonexpert_bytes, m.size_expert16_bytes, m.quant_ratio) == (3_160_000_000, 336_000_000, 4.0)
    assert h.gpu_mem_bytes == 80_000_000_000
    assert h.transfer_bw_bytes_per_s == pytest.approx(12.285e9, rel=1e-4)


def test_builtin_profiles(moe):
    a, _ = moe.load_profiles("[model]\nbuiltin = mixtral-sec41\n")
    assert a == moe.mixtral_sec41()
    b, _ = moe.load_profiles("[model]\nbuiltin = mixtral-table1\n")
    assert b == moe.mixtral_table1()
    assert (b.size_nonexpert_bytes, b.size_expert16_bytes) == (4_090_000_000, 352_031_250)
    with pytest.raises(moe.ValidationError):  # ParseError maps to status 3
        moe.load_profiles("[model]\nbuiltin = nope\n")


def test_overrides_recalibrate(moe):
    m, h = moe.load_profiles("[model]\nbuiltin = mixtral-sec41\nnum_layers = 16\nsize_expert16_bytes = 100MB\n"
                             "[hardware]\ngpu_mem_bytes = 24GB\ntransfer_bw_bytes_per_s = 10GB\n")
    assert m.num_layers == 16 and m.size_expert16_bytes == 100_000_000 and m.quant_ratio == 4.0
    assert m.compute_latency16_s == pytest.approx(0.9 / (13.0 * 16 * 2), rel=1e-12)
    assert h.gpu_mem_bytes == 24_000_000_000 and h.transfer_bw_bytes_per_s == 10e9


@pytest.mark.parametrize("doc", ["[model]\nexperts_per_layer = 0\n", "[model]\ntop_k = 9\n",
                                 "[model]\nquant_ratio = 1.0\n", "[model]\ncompute_penalty4 = 0.5\n",
                                 "[hardware]\ngpu_mem_bytes = 0\n"])
def test_invariant_violations(moe, doc):
    with pytest.raises(moe.ValidationError):
        moe.load_profiles(doc)


@pytest.mark.parametrize("doc", ["num_layers = 3\n", "[model]\nnum_layers\n", "[model]\nwat = 1\n",
                                 "[wat]\nkey = 1\n", "[model\nnum_layers = 3\n", "[model]\nnum_layers = abc\n"])
def test_parse_errors(moe, doc):
    with pytest.raises(moe.MoeError) as ei:
        moe.load_profiles(doc)
    assert ei.value.code == 3


def test_parse_size(moe):
    assert moe.parse_size("30GB") == 30_000_000_000
    assert moe.parse_size("336MB") == 336_000_000
    assert moe.parse_size("84000000") == 84_000_000
    assert moe.parse_size("84000000B") == 84_000_000
    assert moe.parse_size("2.5GB") == 2_500_000_000
    assert moe.parse_size("3.16gb") == 3_160_000_000
    assert moe.parse_size(" 12 GB ") == 12_000_000_000
    for bad in ("30KB", "GB", "-3GB", "12XB", ""):
        with pytest.raises(moe.MoeError):
            moe.parse_size(bad)


def test_expert_and_model_sizes(moe):
    mx = moe.mixtral_sec41()
    assert moe.expert_size(mx, 1) == 336_000_000 and moe.expert_size(mx, 0) == 84_000_000
    odd = moe.mixtral_sec41()
    odd.size_expert16_bytes = 352_031_250
    assert moe.expert_size(odd, 0) == 88_007_812
    t1 = moe.mixtral_table1()
    assert moe.model_size(t1, 256, 0) == 23_552_499_872
    assert moe.model_size(t1, 0, 2) == 94_210_000_000
    assert abs(moe.model_size(t1, 256, 2) - 26_620_000_000) < 50_000_000
    with pytest.raises(moe.ValidationError):
        moe.model_size(t1, 257, 2)
    prev = moe.model_size(mx, 0, 2)
    for n4 in range(1, 257, 17):
        cur = moe.model_size(mx, n4, 2)
        assert cur < prev
        prev = cur


def test_shape_profiles_match_engine_bytes(moe):
    """MoeShape -> exact bytes the engine allocates."""
    p = moe.profile_for_shape(4096, 14336, 32)
    assert moe.expert_size(p, 1) == 352_321_536 and moe.expert_size(p, 0) == 90_832_896
    t = moe.profile_for_shape(512, 1792, 2)
    assert moe.expert_size(t, 1) == 5_505_024 and moe.expert_size(t, 0) == 1_419_264


def test_fingerprint_tracks_fields(moe):
    base = moe.mixtral_sec41()
    fp = moe.profile_fingerprint(base)
    assert fp == 0x212050EE9483C8EF  # SURVEY §8c probe KAT
    for field, val in (("top_k", 3), ("compute_penalty4", 1.2), ("size_expert16_bytes", 336_000_001)):
        c = moe.mixtral_sec41()
        setattr(c, field, val)
        assert moe.profile_fingerprint(c) != fp


# ----------------------------------------------------------- test_planner.cpp
def test_eq1_kats(moe, kM):
    assert moe.num_experts_16(24_000_000_000, kM) == 0
    assert moe.num_experts_16(24_664_000_000, kM) == 0
    assert moe.num_experts_16(30_000_000_000, kM) == 21
    assert moe.num_experts_16(120_000_000_000, kM) == 256


def test_eq1_monotone(moe, kM):
    all4 = kM.size_nonexpert_bytes + 256 * moe.expert_size(kM, 0)
    prev = 0
    for mem in range(1_000_000_000, 130_000_000_001, 499_999_999):
        n16 = moe.num_experts_16(mem, kM)
        assert n16 >= prev
        if mem <= all4:
            assert n16 == 0
        if mem >= all4 + 3 * moe.expert_size(kM, 0):
            assert n16 >= 1
        prev = n16


def test_throughput_plan_30gb(moe, kM):
    plan = moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, 0), hw(moe, 30_000_000_000), kM)
    assert (plan.n4, plan.n_gpu, plan.swap_slot_bytes) == (235, 256, 0)
    assert moe.gpu_footprint(plan, kM) == 29_956_000_000
    assert moe.validate_plan(plan, hw(moe, 30_000_000_000), kM) == []


def test_throughput_plan_20gb(moe, kM):
    plan = moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, 0), hw(moe, 20_000_000_000), kM)
    assert (plan.n4, plan.n_gpu, plan.swap_slot_bytes) == (256, 199, 84_000_000)


def test_infeasible(moe, kM):
    with pytest.raises(moe.InfeasibleError) as ei:
        moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, 0), hw(moe, 2_000_000_000), kM)
    assert ei.value.code == 4


def test_quality_plans(moe, kM):
    all4 = moe.make_plan(moe.TaskRequest(moe.QUALITY, 256, 0), hw(moe, 20_000_000_000), kM)
    assert (all4.n4, all4.n_gpu, all4.swap_slot_bytes) == (256, 199, 84_000_000)
    r16 = moe.make_plan(moe.TaskRequest(moe.QUALITY, 0, 0), hw(moe, 94_000_000_000), kM)
    assert (r16.n4, r16.n_gpu, r16.swap_slot_bytes) == (0, 256, 0)
    assert moe.gpu_footprint(r16, kM) == 89_176_000_000
    p16 = moe.make_plan(moe.TaskRequest(moe.QUALITY, 0, 0), hw(moe, 50_000_000_000), kM)
    assert (p16.n_gpu, p16.swap_slot_bytes) == (138, 336_000_000)
    for n4 in (None, 300):
        with pytest.raises(moe.ValidationError):
            moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 0), hw(moe, 50_000_000_000), kM)


def test_quantization_subset_kat(moe, kM):
    """SURVEY §8a a4 probe KAT: Mixtral n4=8 seed 7."""
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 7), hw(moe, 10**15), kM)
    ids = [(i // 8, i % 8) for i, p in enumerate(plan.precision) if p == 0]
    assert ids == [(1, 7), (10, 5), (11, 2), (13, 4), (21, 6), (24, 2), (26, 1), (27, 6)]


def test_trace_kat(moe, kM):
    """SURVEY §8a a7 probe KATs."""
    slots, _ = moe.generate_trace(kM, 1, 0)
    assert [slots[2 * l:2 * l + 2] for l in range(4)] == [[4, 6], [0, 4], [1, 5], [0, 3]]
    tiny = moe.ModelProfile(num_layers=2, size_expert16_bytes=5_505_024)
    slots, _ = moe.generate_trace(tiny, 4, 0)
    assert slots == [4, 6, 0, 4, 1, 5, 0, 3, 0, 1, 3, 4, 0, 4, 3, 4]


@pytest.mark.parametrize("case", ["fits", "p4_first", "tight", "fixed_point"])
def test_greedy_toy_by_hand(moe, case):
    t = toy(moe)
    P4, P16, GPU, CPU = 0, 1, 0, 1
    if case == "fits":
        p = moe.assign_locations([P4] * 4, hw(moe, 1400), t)
        assert p.n_gpu == 4 and p.swap_slot_bytes == 0
    elif case == "p4_first":
        # test_planner.cpp:157-168 expects (0,0) GPU, (1,0) CPU, swap 400 at a
        # 2000 B budget, but full residency also costs exactly 1000 + 2*100 +
        # 2*400 = 2000 B (no swap needed), and the reference implementation
        # (planner.cpp:88-94, run from oracle/_ref) returns all-resident.  We
        # follow the implementation; one byte less gives the P4-first cut.
        p = moe.assign_locations([P16, P4, P16, P4], hw(moe, 2000), t)
        assert p.location == [GPU] * 4 and p.swap_slot_bytes == 0
        p = moe.assign_locations([P16, P4, P16, P4], hw(moe, 1999), t)
        assert p.location == [CPU, GPU, CPU, GPU] and p.swap_slot_bytes == 400
    elif case == "tight":
        p = moe.assign_locations([P4] * 4, hw(moe, 1300), t)
        assert p.location == [GPU, GPU, CPU, CPU] and p.swap_slot_bytes == 100
    else:
        p = moe.assign_locations([P4, P16, P4, P16], hw(moe, 1600), t)
        assert p.n_gpu == 2 and p.swap_slot_bytes == 400 and moe.gpu_footprint(p, t) == 1600


def test_validate_plan_reports(moe, kM):
    h = hw(moe, 30_000_000_000)
    plan = moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, 0), h, kM)
    tight = hw(moe, moe.gpu_footprint(plan, kM) - 1)
    v = moe.validate_plan(plan, tight, kM)
    assert len(v) == 1 and "exceeds budget" in v[0] and "by 1 B" in v[0]
    plan.location[0] = 1
    v = moe.validate_plan(plan, h, kM)
    assert v and "swap_slot_bytes" in v[0]


def _random_task(moe, rng_next, rng_below):
    pass


def test_property_planner_output_valid(moe, kM):
    """test_planner.cpp:235-264 (1200 cases)."""
    rng = np.random.default_rng(2024)
    produced = 0
    for _ in range(1200):
        budget = 2_000_000_000 + int(rng.integers(0, 98_000_000_000))
        seed = int(rng.integers(0, 2**63))
        task = moe.TaskRequest(moe.THROUGHPUT, None, seed) if rng.integers(0, 2) == 0 else \
            moe.TaskRequest(moe.QUALITY, int(rng.integers(0, 257)), seed)
        try:
            plan = moe.make_plan(task, hw(moe, budget), kM)
        except moe.InfeasibleError:
            continue
        assert moe.validate_plan(plan, hw(moe, budget), kM) == []
        produced += 1
    assert produced >= 1000


def test_property_p4_first(moe, kM):
    """test_planner.cpp:266-280 (1000 cases)."""
    rng = np.random.default_rng(99)
    for _ in range(1000):
        budget = 4_000_000_000 + int(rng.integers(0, 96_000_000_000))
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, int(rng.integers(0, 257)), int(rng.integers(0, 2**63))),
                             hw(moe, budget), kM)
        p4_cpu = any(p == 0 and l == 1 for p, l in zip(plan.precision, plan.location))
        p16_gpu = any(p == 1 and l == 0 for p, l in zip(plan.precision, plan.location))
        assert not (p4_cpu and p16_gpu)


def test_property_throughput_maximal(moe, kM):
    """test_planner.cpp:282-302 (1000 cases; maximality checked on 200)."""
    rng = np.random.default_rng(555)
    s4, s16 = moe.expert_size(kM, 0), moe.expert_size(kM, 1)
    for it in range(1000):
        budget = 3_300_000_000 + int(rng.integers(0, 96_000_000_000))
        plan = moe.make_plan(moe.TaskRequest(moe.THROUGHPUT, None, int(rng.integers(0, 2**63))), hw(moe, budget), kM)
        if plan.n4 < 256:
            assert plan.n_gpu == 256
        if it % 5:
            continue
        base = kM.size_nonexpert_bytes + sum((s16 if p else s4) for p, l in zip(plan.precision, plan.location) if l == 0)
        for i, l in enumerate(plan.location):
            if l != 1:
                continue
            rest = [(s16 if p else s4) for j, (p, ll) in enumerate(zip(plan.precision, plan.location)) if ll == 1 and j != i]
            moved = base + (s16 if plan.precision[i] else s4) + (max(rest) if rest else 0)
            assert moved > budget


def test_property_deterministic(moe, kM):
    rng = np.random.default_rng(31337)
    for _ in range(200):
        budget = 3_300_000_000 + int(rng.integers(0, 90_000_000_000))
        seed = int(rng.integers(0, 2**63))
        task = moe.TaskRequest(moe.THROUGHPUT, None, seed) if rng.integers(0, 2) == 0 else \
            moe.TaskRequest(moe.QUALITY, int(rng.integers(0, 257)), seed)
        a, b = moe.make_plan(task, hw(moe, budget), kM), moe.make_plan(task, hw(moe, budget), kM)
        assert a == b


def test_simulate_calibration_kats(moe, kM):
    """13.00 tps ceiling, ~0.547 all-host floor, toy 146.2 tps."""
    slots, _ = moe.generate_trace(kM, 100, 1)
    gpu16 = moe.assign_locations([1] * 256, hw(moe, 10**15), kM)
    assert moe.simulate(gpu16, slots, 100, kM, hw(moe, 10**15)).throughput_tps == pytest.approx(13.0, abs=0.01)
    cpu16 = moe.PlacementPlan([1] * 256, [1] * 256, 336_000_000)
    r = moe.simulate(cpu16, slots, 100, kM, hw(moe, 10**15))
    assert 0.50 <= r.throughput_tps <= 0.65 and r.hit_rate == 0.0
    t = moe.ModelProfile(num_layers=1, experts_per_layer=2, top_k=1, size_nonexpert_bytes=1,
                         size_expert16_bytes=336_000_000, compute_latency16_s=0.0, nonexpert_latency_s=0.0)
    ts, _ = moe.generate_trace(t, 10, 0)
    r = moe.simulate(moe.PlacementPlan([0, 0], [1, 1], 84_000_000), ts, 10, t, hw(moe, 10**12))
    assert r.throughput_tps == pytest.approx(146.25, abs=0.05)


def test_trace_roundtrip_and_errors(moe, kM):
    slots, fp = moe.generate_trace(kM, 5, 3)
    doc = moe.write_trace(kM, 5, slots)
    tr = moe.read_trace(doc)
    assert tr["slots"] == slots and tr["fingerprint"] == fp and tr["tokens"] == 5
    lines = doc.split("\n")
    bad_dup = "\n".join(lines[:1] + ["0,0,3,3"] + lines[2:])
    bad_range = "\n".join(lines[:1] + ["0,0,3,8"] + lines[2:])
    bad_order = "\n".join(lines[:1] + ["0,0,5,3"] + lines[2:])
    for bad in (bad_dup, bad_range, bad_order, doc + "junk\n", lines[0] + "\n"):
        with pytest.raises(moe.MoeError) as ei:
            moe.read_trace(bad)
        assert ei.value.code == 3


# ----------------------------------------------------------- live vs oracle/_ref
def test_live_plans_match_reference(moe, ref, kM):
    rng = np.random.default_rng(7)
    rp = ref.default_profile(0)
    for _ in range(400):
        budget = int(rng.integers(1_000_000_000, 110_000_000_000))
        pref = int(rng.integers(0, 2))
        n4 = int(rng.integers(0, 257)) if pref else None
        seed = int(rng.integers(0, 2**63))
        st, prec, loc, swap = ref.make_plan(rp, budget, MIX_BW, pref, n4, seed)
        if st != 0:
            with pytest.raises(moe.MoeError) as ei:
                moe.make_plan(moe.TaskRequest(pref, n4, seed), hw(moe, budget), kM)
            assert ei.value.code == st
            continue
        plan = moe.make_plan(moe.TaskRequest(pref, n4, seed), hw(moe, budget), kM)
        assert plan.precision == prec.tolist() and plan.location == loc.tolist() and plan.swap_slot_bytes == swap


def test_live_traces_simulate_match_reference(moe, ref):
    rng = np.random.default_rng(11)
    for L, E, k in ((32, 8, 2), (2, 8, 2), (4, 16, 4), (3, 4, 4)):
        prof = moe.ModelProfile(num_layers=L, experts_per_layer=E, top_k=k)
        rp = ref.profile(prof)
        for _ in range(10):
            seed = int(rng.integers(0, 2**63))
            st, rslots, rfp = ref.generate_trace(prof, 37, seed)
            slots, fp = moe.generate_trace(prof, 37, seed)
            assert st == 0 and slots == rslots.tolist() and fp == rfp
            assert moe.write_trace(prof, 37, slots) == ref.write_trace(prof, 37, rslots)
            budget = int(rng.integers(1_000_000_000, 100_000_000_000))
            st, prec, loc, swap = ref.make_plan(rp, budget, MIX_BW, 1, int(rng.integers(0, L * E + 1)), seed)
            if st != 0:
                continue
            plan = moe.PlacementPlan(prec.tolist(), loc.tolist(), swap)
            for lru in (0, 1, 3):
                st, sim = ref.simulate(prof, MIX_BW, prec, loc, swap, 37, rslots, lru)
                r = moe.simulate(plan, slots, 37, prof, hw(moe, budget), lru)
                assert [r.activations, r.hits, r.bytes_transferred, r.transfer_ns, r.compute_ns,
                         r.nonexpert_ns] == sim.tolist()
            assert moe.expected_throughput(plan, prof, hw(moe, budget)) == ref.expected_throughput(prof, MIX_BW, prec, loc, swap)


def test_live_load_profiles_match_reference(moe, ref):
    docs = ["", "[model]\nbuiltin = mixtral-table1\n", "[model]\nnum_layers = 24\n[hardware]\ngpu_mem_bytes = 48GB\n",
            "# c\n; c\n[model]\n top_k = 3 \nquant_ratio=3.5\n[hardware]\ntransfer_bw_bytes_per_s = 12.5e9\n",
            "[model]\ncompute_latency16_s = 0.001\nnonexpert_latency_s=0.01\n[quality]\ndataset = x\n"]
    for doc in docs:
        st, rp, mem, bw = ref.load_profiles(doc)
        m, h = moe.load_profiles(doc)
        assert st == 0
        assert (m.num_layers, m.experts_per_layer, m.top_k, m.size_nonexpert_bytes, m.size_expert16_bytes,
                m.quant_ratio, m.compute_latency16_s, m.compute_penalty4, m.nonexpert_latency_s) == \
               (rp.num_layers, rp.experts_per_layer, rp.top_k, rp.size_nonexpert_bytes, rp.size_expert16_bytes,
                rp.quant_ratio, rp.compute_latency16_s, rp.compute_penalty4, rp.nonexpert_latency_s)
        assert (h.gpu_mem_bytes, h.transfer_bw_bytes_per_s) == (mem, bw)


# ----------------------------------------------------------- plan artifact (serialize.cpp)
def _plan_mutations(doc):
    """Malformed / mismatched variants of a plan document, each rejected by
    serialize.cpp:119-149 (ParseError or ValidationError)."""
    import json
    j = json.loads(doc)
    out = [doc.replace("moeserve.plan.v1", "moeserve.plan.v2"), doc.replace('"format"', '"fmt"'),
           "", "[]", "{", doc[: len(doc) // 2]]
    fp = j["profile_fingerprint"]
    out.append(doc.replace(fp, fp[:-1] + ("0" if fp[-1] != "0" else "1")))
    for fn in (lambda e: e.pop(),                              # missing expert
               lambda e: e.append(list(e[0])),                 # duplicate
               lambda e: e[0].__setitem__(2, "p8"),            # unknown precision
               lambda e: e[0].__setitem__(3, "disk"),          # unknown location
               lambda e: e[0].pop(),                           # short row
               lambda e: e[1].__setitem__(1, 99),              # slot out of range
               lambda e: e[1].__setitem__(0, -1)):             # layer out of range
        jj = json.loads(doc)
        fn(jj["experts"])
        out.append(json.dumps(jj))
    return out


def test_plan_json_roundtrip_and_errors(moe, kM):
    plan = moe.make_plan(moe.TaskRequest(1, 100, 9), hw(moe, 40_000_000_000), kM)
    doc = moe.write_plan(plan, kM)
    assert doc.startswith('{\n  "format": "moeserve.plan.v1",\n') and doc.endswith("\n  ]\n}\n")
    assert moe.read_plan(doc, kM) == plan
    import json
    assert moe.read_plan(json.dumps(json.loads(doc)), kM) == plan  # any JSON layout of the schema
    for bad in _plan_mutations(doc):
        with pytest.raises(moe.MoeError) as ei:
            moe.read_plan(bad, kM)
        assert ei.value.code == 3, bad[:80]
    with pytest.raises(moe.ValidationError):  # a plan for another profile
        moe.read_plan(doc, moe.mixtral_table1())


def test_live_plan_json_matches_reference(moe, ref, kM):
    if not ref.has_serialize:
        pytest.skip("oracle/_ref built without serialize.cpp (no nlohmann/json)")
    rng = np.random.default_rng(11)
    rp = ref.default_profile(0)
    for _ in range(40):
        budget = int(rng.integers(1_000_000_000, 110_000_000_000))
        n4 = int(rng.integers(0, 257))
        seed = int(rng.integers(0, 2**64, dtype=np.uint64))
        st, prec, loc, swap = ref.make_plan(rp, budget, MIX_BW, 1, n4, seed)
        if st != 0:
            continue
        plan = moe.PlacementPlan(prec.tolist(), loc.tolist(), swap, seed)
        wst, rdoc = ref.write_plan(rp, prec, loc, seed, swap)
        assert wst == 0
        doc = moe.write_plan(plan, kM)
        assert doc == rdoc  # byte-identical to nlohmann dump(2)
        rst, rprec, rloc, rseed, rswap = ref.read_plan(doc, rp)
        assert rst == 0 and rprec.tolist() == plan.precision and rloc.tolist() == plan.location
        assert (rseed, rswap) == (seed, swap)
        for bad in _plan_mutations(doc):
            rst = ref.read_plan(bad, rp)[0]
            with pytest.raises(moe.MoeError) as ei:
                moe.read_plan(bad, kM)
            assert ei.value.code == rst, bad[:80]
    # toy profile, empty-layer edge: 2x2 experts
    tp = toy(moe)
    rtp = ref.profile(tp)
    plan = moe.PlacementPlan([0, 1, 1, 0], [1, 0, 1, 0], 400, 0)
    assert moe.write_plan(plan, tp) == ref.write_plan(rtp, plan.precision, plan.location, 0, 400)[1]


# ----------------------------------------------------------- pareto (f3)
def _csv_restated(rows, measured=None):
    """cli.cpp:253-270 restated over reference rows (+ the measured columns)."""
    g = lambda v: "%.10g" % v  # format_double, serialize.cpp:93-97
    out = ("budget_bytes,n4,n_gpu,gpu_bytes,throughput_tps,hit_rate,bytes_transferred,ppl_estimate,on_frontier,"
           "status" + (",measured_tps,measured_hit_rate" if measured is not None else "") + "\n")
    for i, r in enumerate(rows):
        out += f"{int(r['budget'])},{int(r['n4'])},"
        if r["feasible"]:
            tot = (int(r["transfer_ns"]) + int(r["compute_ns"]) + int(r["nonexpert_ns"])) / 1e9
            hit = 1.0 if r["activations"] == 0 else int(r["hits"]) / int(r["activations"])
            out += (f"{int(r['n_gpu'])},{int(r['gpu_bytes'])},{g(int(r['tokens']) / tot)},{g(hit)},"
                    f"{int(r['bytes_transferred'])},{g(float(r['ppl']))},{int(r['on_frontier'])},ok")
        else:
            out += f"-,-,-,-,-,{g(float(r['ppl']))},0,infeasible"
        if measured is not None:
            m = measured[i]
            out += ",-,-" if (m is None or not r["feasible"]) else f",{g(m[0])},{g(m[1])}"
        out += "\n"
    return out


def test_live_pareto_sweep_matches_reference(moe, ref, kM):
    rng = np.random.default_rng(1407)
    rp = ref.default_profile(0)
    for case in range(6):
        budgets = sorted(int(v) for v in rng.integers(3_000_000_000, 100_000_000_000, size=int(rng.integers(1, 7))))
        grid = [int(v) for v in rng.integers(0, 257, size=int(rng.integers(1, 5)))]
        seed = int(rng.integers(0, 2**63))
        name = ("wikitext2", "ptb", "c4")[case % 3]
        st, p16, p4 = ref.builtin_anchors(name)
        a = moe.builtin_anchors(name)
        assert st == 0 and (a.ppl_all16, a.ppl_all4) == (p16, p4)
        st, rrows = ref.pareto_sweep(rp, MIX_BW, budgets, grid, 60, seed, p16, p4)
        assert st == 0
        rows = moe.pareto_sweep(budgets, grid, kM, hw(moe, 1), 60, seed, a)
        assert len(rows) == len(rrows)
        for r, q in zip(rows, rrows):
            assert (r.budget, r.n4, r.feasible, r.on_frontier, r.ppl) == \
                (q["budget"], q["n4"], bool(q["feasible"]), bool(q["on_frontier"]), q["ppl"])
            if r.feasible:
                assert (r.n_gpu, r.gpu_bytes) == (q["n_gpu"], q["gpu_bytes"])
                rep = r.report
                assert [rep.tokens, rep.activations, rep.hits, rep.bytes_transferred, rep.transfer_ns, rep.compute_ns,
                        rep.nonexpert_ns] == [int(q[k]) for k in ("tokens", "activations", "hits", "bytes_transferred",
                                                                   "transfer_ns", "compute_ns", "nonexpert_ns")]
        assert moe.pareto_csv(rows) == _csv_restated(rrows)
        meas = [None if i % 2 else (123.25 + i, 0.5) for i in range(len(rows))]
        assert moe.pareto_csv(rows, meas) == _csv_restated(rrows, meas)


def test_live_pareto_primitives_match_reference(moe, ref):
    rng = np.random.default_rng(3)
    for _ in range(200):  # frontier over random point clouds with ties
        n = int(rng.integers(0, 40))
        tps = rng.integers(0, 6, n).astype(np.float64)
        ppl = rng.integers(0, 4, n) * 0.5 + 3.0
        gb = rng.integers(0, 5, n).astype(np.int64)
        st, mask = ref.frontier_mask(tps, ppl, gb)
        assert st == 0 and moe.frontier_mask(tps.tolist(), ppl.tolist(), gb.tolist()) == mask.tolist()
    anchors = [(3.81, 4.0), (13.59, 14.17), (7.24, 7.4), (5.0, 5.0), (0.5, 4.0), (4.0, 3.0), (1.0, 2.0)]
    for p16, p4 in anchors:
        for n4, num_e in ((0, 256), (77, 256), (256, 256), (257, 256), (-1, 8), (3, 0)):
            st, v = ref.ppl_estimate(n4, p16, p4, num_e)
            if st:
                with pytest.raises(moe.MoeError) as ei:
                    moe.ppl_estimate(n4, moe.QualityAnchors(p16, p4), num_e)
                assert ei.value.code == st
            else:
                assert moe.ppl_estimate(n4, moe.QualityAnchors(p16, p4), num_e) == v
        for budget in (3.0, p16, (p16 + p4) / 2, p4, p4 + 1):
            st, v = ref.n4_for_budget(budget, p16, p4, 256)
            if st:
                with pytest.raises(moe.MoeError) as ei:
                    moe.n4_for_budget(budget, moe.QualityAnchors(p16, p4), 256)
                assert ei.value.code == st
            else:
                assert moe.n4_for_budget(budget, moe.QualityAnchors(p16, p4), 256) == v
    docs = ["", "[quality]\ndataset = ptb\n", "[quality]\ndataset = mine\nppl_all16 = 5\nppl_all4 = 6\n",
            "[quality]\nppl_all4 = 3.9\n", "[quality]\nppl_all4 = 3.0\n", "[quality]\nfoo = 1\n",
            "[quality]\nppl_all16 = x\n", "[model]\ntop_k = 2\n[quality]\ndataset = c4\n"]
    for doc in docs:
        st, a, b = ref.load_anchors(doc, 3.81, 4.0)
        if st:
            with pytest.raises(moe.MoeError) as ei:
                moe.load_anchors(doc)
            assert ei.value.code == st, doc
        else:
            got = moe.load_anchors(doc)
            assert (got.ppl_all16, got.ppl_all4) == (a, b), doc
    with pytest.raises(moe.UsageError):
        moe.builtin_anchors("imagenet")


def test_pareto_cli_parsing_and_unmeasured_sweep(moe):
    from paper_2407_14417_b200 import pareto
    assert pareto.parse_mem_range(moe, "24GB:30GB:2GB") == [24 * 10**9, 26 * 10**9, 28 * 10**9, 30 * 10**9]
    assert pareto.parse_mem_range(moe, "1GB") == [10**9]
    for bad in ("1GB:2GB", "2GB:1GB:1GB", "1GB:2GB:0", "x"):
        with pytest.raises(moe.MoeError):
            pareto.parse_mem_range(moe, bad)
    assert pareto.parse_n4_grid(moe, "0,5,256") == [0, 5, 256]
    for bad in ("", "1,,2", "-1", "a"):
        with pytest.raises(moe.UsageError):
            pareto.parse_n4_grid(moe, bad)
    rows, meas = pareto.measured_sweep(moe, [10**9, 5 * 10**9], [0, 16], (2, 8, 2, 512, 1792), 12.285e9, 20,
                                       measure=False)
    assert len(rows) == 4 and meas == [None] * 4
    doc = moe.pareto_csv(rows, meas)
    assert doc.splitlines()[0].endswith(",status,measured_tps,measured_hit_rate")
