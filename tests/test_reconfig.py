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
