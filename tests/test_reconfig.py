"""Reconfiguration: diff_plans / estimate_cost / apply.

The reference has no reconfig test suite. These tests compare with the
reference library compiled from /root/reference (oracle/_ref): action lists,
costs and replays on seeded random plan pairs, plus corrupted action lists
(reconfig.cpp:84-168 error cases).  The GPU tests (test_gpu_engine.py) run the
executor, MoeEngine.reconfigure.
"""
import numpy as np
import pytest

MIX_BW = 336_000_000.0 / 0.02735


def _plans(moe, prof, rng):
    a = moe.make_plan(moe.TaskRequest(1, int(rng.integers(0, 257)), int(rng.integers(0, 2**32))),
                      moe.HardwareProfile(int(rng.integers(4, 100)) * 10**9, MIX_BW), prof)
    b = moe.make_plan(moe.TaskRequest(1, int(rng.integers(0, 257)), int(rng.integers(0, 2**32))),
                      moe.HardwareProfile(int(rng.integers(4, 100)) * 10**9, MIX_BW), prof)
    return a, b


def test_diff_apply_roundtrip_and_grouping(moe):
    prof = moe.mixtral_sec41()
    rng = np.random.default_rng(1)
    for _ in range(20):
        a, b = _plans(moe, prof, rng)
        acts, nbytes, t = moe.diff_plans(a, b, prof, moe.HardwareProfile(1, MIX_BW))
        kinds = [k for k, *_ in acts]
        # releasing group (Offload, Quantize) before consuming (Dequantize, Fetch)
        first_consuming = next((i for i, k in enumerate(kinds) if k in (moe.FETCH, moe.DEQUANTIZE)), len(kinds))
        assert all(k in (moe.OFFLOAD, moe.QUANTIZE) for k in kinds[:first_consuming])
        assert all(k in (moe.FETCH, moe.DEQUANTIZE) for k in kinds[first_consuming:])
        assert t == pytest.approx(nbytes / MIX_BW, rel=1e-15)
        c = moe.apply_reconfig(a, acts, b.seed, prof)
        assert (c.precision, c.location, c.seed) == (b.precision, b.location, b.seed)
        assert c.swap_slot_bytes == b.swap_slot_bytes
        assert moe.diff_plans(a, a, prof, moe.HardwareProfile(1))[:2] == ([], 0)


def test_apply_rejects_inconsistent_lists(moe):
    prof = moe.mixtral_sec41()
    a, b = _plans(moe, prof, np.random.default_rng(2))
    acts, _, _ = moe.diff_plans(a, b, prof, moe.HardwareProfile(1))
    assert acts
    bad = [acts + [acts[0]],                                        # an expert acted on twice
           [(moe.FETCH if acts[0][0] == moe.OFFLOAD else moe.OFFLOAD,) + tuple(acts[0][1:])] + acts[1:]]
    k, l, s, p, loc = acts[0]
    bad.append([(k, l, s, p, 1 - loc if k in (moe.OFFLOAD, moe.FETCH) else loc)] + acts[1:]
               if k in (moe.OFFLOAD, moe.FETCH) else [(k, l, s, 1 - p, loc)] + acts[1:])
    for lst in bad:
        with pytest.raises(moe.ValidationError):
            moe.apply_reconfig(a, lst, b.seed, prof)


def test_live_reconfig_matches_reference(moe, ref):
    prof = moe.mixtral_sec41()
    rp = ref.default_profile(0)
    rng = np.random.default_rng(2407)
    for case in range(60):
        a, b = _plans(moe, prof, rng)
        b.seed = int(rng.integers(0, 2**63))
        acts, nbytes, t = moe.diff_plans(a, b, prof, moe.HardwareProfile(1, MIX_BW))
        st, racts, rbytes, rt = ref.reconfig_diff(rp, MIX_BW, a.precision, a.location, b.precision, b.location, b.seed)
        assert st == 0 and acts == racts and nbytes == rbytes and t == rt
        # replay under random budgets (mid-sequence and final checks) and corrupted lists
        budget = int(rng.integers(3, 100)) * 10**9
        variants = [acts, acts[::-1], acts[1:], acts + acts[:1]]
        for lst in variants:
            for bud in (0, budget):
                st, p_, l_, sw, sd = ref.reconfig_apply(rp, a.precision, a.location, a.seed, lst, b.seed, bud)
                if st:
                    with pytest.raises(moe.MoeError) as ei:
                        moe.apply_reconfig(a, lst, b.seed, prof, moe.HardwareProfile(bud, MIX_BW) if bud else None)
                    assert ei.value.code == st
                else:
                    c = moe.apply_reconfig(a, lst, b.seed, prof, moe.HardwareProfile(bud, MIX_BW) if bud else None)
                    assert (c.precision, c.location, c.swap_slot_bytes, c.seed) == (p_.tolist(), l_.tolist(), sw, sd)


# ----------------------------------------------------------- artifacts (serialize.cpp:160-243)
def _reconfig_mutations(doc):
    import json
    j = json.loads(doc)
    out = [doc.replace("moeserve.reconfig.v1", "moeserve.plan.v1"), doc + "x", "{}", doc[:-3]]
    fp = j["profile_fingerprint"]
    out.append(doc.replace(fp, "0" * len(fp)))
    if j["actions"]:
        for fn in (lambda a: a[0].__setitem__(0, "teleport"), lambda a: a[0].__setitem__(1, 99),
                   lambda a: a[0].__setitem__(3, "p8"), lambda a: a[0].pop(), lambda a: a[0].__setitem__(1, "0"),
                   lambda a: a[0].__setitem__(2, 1.75), lambda a: a[0].__setitem__(0, 3)):
            jj = json.loads(doc)
            fn(jj["actions"])
            out.append(json.dumps(jj))
    jj = json.loads(doc)
    jj["bytes_moved"] += 1
    out.append(json.dumps(jj))
    jj = json.loads(doc)
    jj["target_seed"] = "7"
    out.append(json.dumps(jj))
    return out


def test_live_reconfig_artifact_matches_reference(moe, ref):
    if not ref.has_serialize:
        pytest.skip("oracle/_ref built without serialize.cpp (no nlohmann/json)")
    prof = moe.mixtral_sec41()
    rp = ref.default_profile(0)
    rng = np.random.default_rng(77)
    for case in range(25):
        a, b = _plans(moe, prof, rng)
        b.seed = int(rng.integers(0, 2**64, dtype=np.uint64))
        bw = float(rng.choice([MIX_BW, 55.6e9, 1e9 / 3, 7.5e12]))
        hw = moe.HardwareProfile(1, bw)
        acts, _, _ = moe.diff_plans(a, b, prof, hw)
        st, rdoc = ref.write_reconfig(rp, bw, a.precision, a.location, b.precision, b.location, b.seed)
        doc = moe.write_reconfig(acts, b.seed, prof, hw)
        assert st == 0 and doc == rdoc  # byte-identical, doubles included
        got = moe.read_reconfig(doc, prof, hw)
        rst, racts, rseed, rbytes, rt = ref.read_reconfig(doc, rp, bw)
        assert rst == 0 and got == (racts, rseed, rbytes, rt)
        for bad in _reconfig_mutations(doc):
            rst = ref.read_reconfig(bad, rp, bw)[0]
            if rst == 0:
                assert moe.read_reconfig(bad, prof, hw) == ref.read_reconfig(bad, rp, bw)[1:]
                continue
            with pytest.raises(moe.MoeError) as ei:
                moe.read_reconfig(bad, prof, hw)
            assert ei.value.code == rst, bad[:120]


def test_live_report_text_matches_reference(moe, ref):
    if not ref.has_serialize:
        pytest.skip("oracle/_ref built without serialize.cpp (no nlohmann/json)")
    rng = np.random.default_rng(5)
    cases = [[0, 0, 0, 0, 0, 0, 0], [1, 0, 0, 0, 0, 0, 0], [37, 74, 74, 0, 0, 12345, 1]]
    for _ in range(200):
        tok = int(rng.integers(1, 5000))
        act = int(rng.integers(0, 64 * tok))
        scale = 10 ** int(rng.integers(0, 13))
        cases.append([tok, act, int(rng.integers(0, act + 1)), int(rng.integers(0, 10**13)),
                      int(rng.integers(0, scale)), int(rng.integers(0, scale)), int(rng.integers(0, 10**9))])
    for c in cases:
        r = moe.SimReport(*c)
        for js in (False, True):
            assert moe.report_text(r, js) == ref.report_text(c, js), (c, js)


def test_plan_reader_type_semantics_match_reference(moe, ref):
    """nlohmann get<int>() converts floats / booleans and type-errors on
    strings (exit 1); seeds use the full uint64 range."""
    if not ref.has_serialize:
        pytest.skip("oracle/_ref built without serialize.cpp (no nlohmann/json)")
    import json
    prof = moe.mixtral_sec41()
    rp = ref.default_profile(0)
    plan = moe.make_plan(moe.TaskRequest(1, 100, 9), moe.HardwareProfile(40 * 10**9), prof)
    plan.seed = 2**64 - 5
    doc = moe.write_plan(plan, prof)
    assert moe.read_plan(doc, prof).seed == 2**64 - 5
    variants = []
    for edit in (lambda j: j["experts"][0].__setitem__(1, 0.9), lambda j: j["experts"][0].__setitem__(1, "0"),
                 lambda j: j["experts"][1].__setitem__(1, True), lambda j: j.__setitem__("seed", "1"),
                 lambda j: j.__setitem__("seed", -1), lambda j: j.__setitem__("swap_slot_bytes", 1.5e3),
                 lambda j: j["experts"][0].__setitem__(2, 4)):
        j = json.loads(doc)
        edit(j)
        variants.append(json.dumps(j))
    variants += [doc.replace('"seed": ', '"seed": +'), doc.replace('"seed": ', '"seed": 0'), doc + " \n\t"]
    for v in variants:
        rst, prec, loc, seed, swap = ref.read_plan(v, rp)
        if rst:
            with pytest.raises(moe.MoeError) as ei:
                moe.read_plan(v, prof)
            assert ei.value.code == rst, v[:100]
        else:
            got = moe.read_plan(v, prof)
            assert (got.precision, got.location, got.seed, got.swap_slot_bytes) == (prec.tolist(), loc.tolist(), seed, swap)
