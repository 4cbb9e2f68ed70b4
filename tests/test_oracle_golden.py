"""Pin the oracle before trusting it (CPU only).

1. generator_kat.json: the synthetic-tensor generator (shared contract of the
   oracle and the GPU engine) is pinned by hashes.
2. tiny_moe_hf.npz: the oracle's router / permutation / SwiGLU FFN / combine
   reproduce HF transformers 5.5.0 MixtralSparseMoeBlock (fp32) on the same
   weights -- the semantics the reference's paper ran and the
   source of the north star's MoE-layer math (the reference itself has no
   tensor math).
3. reference_kat.json: plans / traces / simulate counters from the reference
   library compiled from /root/reference match the product's host library.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from helpers import RTOL_BF16, assert_close, bf16_to_f32

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
L, E, K, D, F, SEED, T = 2, 8, 2, 512, 1792, 42, 32
PREC = [[1, 1, 1, 0, 0, 0, 0, 1], [0, 1, 0, 1, 0, 1, 1, 0]]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_generator_kat(orc):
    kat = json.load(open(os.path.join(GOLD, "generator_kat.json")))
    assert [str(orc.L.orc_rand64(42, 7, i)) for i in range(8)] == kat["rand64_seed42_uid7"]
    assert {str(k): orc.weight_shift(k) for k in (512, 1792, 4096, 14336)} == kat["weight_shift"]
    m = orc.model(L, E, K, D, F, SEED)
    gu, dn = orc.expert_bf16(m, 3)
    qgu, sgu, qd, sd = orc.expert_int4(m, 3)
    assert sha(gu) == kat["expert3_bf16_gate_up_sha256"] and sha(dn) == kat["expert3_bf16_down_sha256"]
    assert sha(qgu) == kat["expert3_int4_q_gate_up_sha256"] and sha(sgu) == kat["expert3_int4_s_gate_up_sha256"]
    assert sha(qd) == kat["expert3_int4_q_down_sha256"] and sha(sd) == kat["expert3_int4_s_down_sha256"]
    assert sha(orc.router_weights(m, 1)) == kat["router_layer1_sha256"]
    assert sha(orc.step_input(m, 5, 3)) == kat["step5_input_sha256"]


def test_tiny_plan_kat(moe):
    """assign_quantization(8, tiny, seed 1) -> 4/4 per layer."""
    prof = moe.profile_for_shape(D, F, L, E, K)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    assert [plan.precision[l * E:(l + 1) * E] for l in range(L)] == PREC


@pytest.mark.parametrize("layer", [0, 1])
def test_oracle_matches_hf_mixtral_block(orc, layer):
    z = np.load(os.path.join(GOLD, "tiny_moe_hf.npz"))
    m = orc.model(L, E, K, D, F, SEED)
    x = z["x0"] if layer == 0 else z["oracle_out_0"]
    wg = orc.router_weights(m, layer)
    idx, w, lg = orc.gate_topk(x, wg, T, D, E, K)
    np.testing.assert_allclose(lg, z[f"hf_logits_{layer}"], rtol=1e-5, atol=1e-6)
    assert np.array_equal(idx, z[f"hf_idx_{layer}"])  # HF orders top-k by descending prob == logit
    np.testing.assert_allclose(w, z[f"hf_w_{layer}"], rtol=1e-5, atol=1e-7)
    counts, offsets, perm, inv = orc.permute(idx, T, E, K)
    y = np.zeros((T * K, D), np.float32)
    for s in range(E):
        lo, hi = offsets[s], offsets[s + 1]
        if lo == hi:
            continue
        xs = x[perm[lo:hi] // K]
        if PREC[layer][s] == 1:
            gu, dn = orc.expert_bf16(m, layer * E + s)
            y[lo:hi] = orc.ffn_bf16(xs, hi - lo, gu, dn, D, F)
        else:
            y[lo:hi] = orc.ffn_int4(xs, hi - lo, *orc.expert_int4(m, layer * E + s), D, F)
    moe_out = orc.combine(y, inv, w, None, T, D, K)
    assert_close(bf16_to_f32(moe_out), z[f"hf_out_{layer}"], RTOL_BF16, f"oracle vs HF layer {layer}")
    # the stored whole-layer oracle output (with residual) is reproducible
    out, _, _, _ = orc.moe_layer(m, layer, PREC[layer], x, T)
    assert np.array_equal(out, z[f"oracle_out_{layer}"])


def test_dequant_is_exact_product(orc):
    rows, cols = 4, 256
    w = orc.synth_weight(1, 2, rows * cols, 8).reshape(rows, cols)
    q, s = orc.quantize(w, rows, cols)
    deq = orc.dequant(q, s, rows, cols)
    sf = bf16_to_f32(s)
    for r in range(rows):
        for c in range(0, cols, 37):
            word = int(q[r, c // 8])
            j = c % 8
            qv = ((word >> (4 * (j // 2) + 16 * (j % 2))) & 15) - 8
            assert deq[r, c] == np.float32(qv) * sf[r, c // 128]
    # round-to-nearest quantisation error bound: |w - q*s| <= s/2 (+ clamp)
    err = np.abs(bf16_to_f32(w) - deq)
    assert (err <= np.repeat(sf, 128, axis=1) * 0.5 + 1e-12).all()


def test_reference_kat_planner_and_simulator(moe):
    kat = json.load(open(os.path.join(GOLD, "reference_kat.json")))
    prof = moe.mixtral_sec41()
    assert hex(moe.profile_fingerprint(prof)) == kat["fingerprint"]
    bw = 336_000_000.0 / 0.02735
    for c in kat["cases"]:
        task = moe.TaskRequest(c["preference"], c["n4"], int(c["seed"]))
        hw = moe.HardwareProfile(c["budget"], bw)
        if c["status"] != 0:
            with pytest.raises(moe.MoeError) as ei:
                moe.make_plan(task, hw, prof)
            assert ei.value.code == c["status"]
            continue
        plan = moe.make_plan(task, hw, prof)
        assert "".join(map(str, plan.precision)) == c["precision"]
        assert "".join(map(str, plan.location)) == c["location"]
        assert plan.swap_slot_bytes == c["swap"]
        slots, _ = moe.generate_trace(prof, 50, c["trace_seed"])
        assert sha(np.array(slots, np.int32)) == c["trace_sha256"]
        r = moe.simulate(plan, slots, 50, prof, hw)
        assert [r.activations, r.hits, r.bytes_transferred, r.transfer_ns, r.compute_ns, r.nonexpert_ns] == c["sim"]
        assert moe.expected_throughput(plan, prof, hw) == c["expected_tps"]
        if "plan_json_sha256" in c:  # serialize.cpp:99-117, byte for byte
            plan.seed = int(c["seed"])
            doc = moe.write_plan(plan, prof)
            assert hashlib.sha256(doc.encode()).hexdigest() == c["plan_json_sha256"]
            assert moe.read_plan(doc, prof) == plan


def test_rmsnorm_pinned_order(orc):
    """orc_rmsnorm restated in numpy with the same pinned reduction order
    (per-thread fmaf chains over x[c*256+i]^2, pairwise tree, IEEE 1/sqrt)."""
    import numpy as np
    rng = np.random.default_rng(5)
    for d in (512, 4096, 768):
        x = (rng.integers(-64, 65, size=(3, d)) / 64.0).astype(np.float32)
        xb = (x.view(np.uint32) >> 16).astype(np.uint16)
        got = orc.rmsnorm(xb, 3, d, 1e-5)
        for t in range(3):
            xf = ((xb[t].astype(np.uint32)) << 16).view(np.float32)
            part = np.zeros(256, np.float32)
            for i in range(256):
                acc = np.float32(0)
                for c in range((d - i + 255) // 256):
                    v = xf[c * 256 + i]
                    acc = np.float32(np.float64(v) * v + acc)  # fmaf: exact product, one rounding
                part[i] = acc
            s2 = 128
            while s2 >= 1:
                part[:s2] = part[:s2] + part[s2:2 * s2]
                s2 //= 2
            rstd = np.float32(1.0) / np.sqrt(np.float32(part[0] / np.float32(d) + np.float32(1e-5)))
            ref = xf * rstd
            refb = ((ref.view(np.uint32) + 0x7FFF + ((ref.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16)
            assert np.array_equal(got[t], refb), d
