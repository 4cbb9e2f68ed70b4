"""K1-K5 parity: the sm_100a kernels through the C ABI vs the CPU oracle.

Integer outputs (routing indices, router logits, permutation, histogram,
quantised weights, synthetic tensors) must be bit-exact; fp outputs within
the tolerances in tests/helpers.py.
"""
import numpy as np
import pytest

from helpers import RTOL_BF16, RTOL_F32, RTOL_WEIGHTS, assert_close, bf16_to_f32, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_mod(cuda):
    import torch
    return torch


def test_synth_weight_bitexact(moe, orc, torch_mod, cuda):
    torch = torch_mod
    for n, shift, uid in [(1, 11, 5), (1000, 12, 17), (2 * 1792 * 512 + 3, 12, (3 << 4) | 1)]:
        out = torch.empty(n, dtype=torch.int16, device=cuda)
        moe.synth_weight_bf16(7, uid, n, shift, out)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(out, np.uint16), orc.synth_weight(7, uid, n, shift))
    for K in (512, 1792, 4096, 14336):
        assert moe.weight_shift(K) == orc.weight_shift(K)


@pytest.mark.parametrize("rows,cols", [(16, 128), (32, 512), (64, 1792), (48, 4096)])
def test_quantize_bitexact(moe, orc, torch_mod, cuda, rows, cols):
    """GPU quantiser (fragment-block output) == oracle RTN quantiser, packed."""
    torch = torch_mod
    w = orc.synth_weight(3, 99 + rows, rows * cols, orc.weight_shift(cols)).reshape(rows, cols)
    w[1, :128] = 0  # all-zero group -> scale 1.0
    q_ref, s_ref = orc.quantize(w, rows, cols)
    qb_ref, sb_ref = orc.pack_int4_blocks(q_ref, s_ref, rows, cols)
    wd = to_dev(w, torch, cuda)
    q = torch.empty(rows * cols // 8, dtype=torch.int32, device=cuda)
    s = torch.empty(rows * cols // 128, dtype=torch.int16, device=cuda)
    moe.quantize_g128(wd, rows, cols, q, s)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(q, np.uint32), qb_ref)
    assert np.array_equal(to_np(s, np.uint16), sb_ref)


@pytest.mark.parametrize("rows,cols", [(16, 128), (48, 1792), (32, 4096)])
def test_pack_bf16_blocks_bitexact(moe, orc, torch_mod, cuda, rows, cols):
    torch = torch_mod
    w = orc.synth_weight(5, rows, rows * cols, 9)
    out = torch.empty(rows * cols, dtype=torch.int16, device=cuda)
    moe.pack_bf16_blocks(to_dev(w, torch, cuda), rows, cols, out)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(out, np.uint16), orc.pack_bf16_blocks(w, rows, cols))


@pytest.mark.parametrize("T,d,E,k", [(1, 512, 8, 2), (32, 512, 8, 2), (5, 4096, 8, 2), (257, 4096, 8, 2),
                                     (3, 1024, 16, 4), (2, 768, 64, 8), (1, 256, 2, 1)])
def test_gate_topk_bitexact(moe, orc, torch_mod, cuda, T, d, E, k):
    torch = torch_mod
    x = orc.synth_input(11, 1000 + T, T * d).reshape(T, d)
    wg = orc.synth_weight(11, 2000 + E, E * d, orc.weight_shift(d)).reshape(E, d)
    idx_ref, w_ref, lg_ref = orc.gate_topk(x, wg, T, d, E, k)
    idx = torch.empty(T * k, dtype=torch.int32, device=cuda)
    w = torch.empty(T * k, dtype=torch.float32, device=cuda)
    lg = torch.empty(T * E, dtype=torch.float32, device=cuda)
    moe.gate_topk(to_dev(x, torch, cuda), to_dev(wg, torch, cuda), T, d, E, k, idx, w, lg)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(lg, np.float32).reshape(T, E).view(np.uint32), lg_ref.view(np.uint32)), "logits not bit-exact"
    assert np.array_equal(to_np(idx, np.int32).reshape(T, k), idx_ref)
    np.testing.assert_allclose(to_np(w, np.float32).reshape(T, k), w_ref, rtol=RTOL_WEIGHTS, atol=1e-7)


def test_gate_topk_ties_lower_index(moe, orc, torch_mod, cuda):
    torch = torch_mod
    T, d, E, k = 4, 256, 8, 2
    x = np.full((T, d), 0x3F80, np.uint16)            # 1.0
    wg = np.zeros((E, d), np.uint16)                  # all logits 0 -> ties everywhere
    wg[5, :] = 0x3C00                                 # expert 5 wins, then ties among the rest
    idx_ref, _, _ = orc.gate_topk(x, wg, T, d, E, k)
    assert (idx_ref[:, 0] == 5).all() and (idx_ref[:, 1] == 0).all()
    idx = torch.empty(T * k, dtype=torch.int32, device=cuda)
    w = torch.empty(T * k, dtype=torch.float32, device=cuda)
    moe.gate_topk(to_dev(x, torch, cuda), to_dev(wg, torch, cuda), T, d, E, k, idx, w, None)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(idx, np.int32).reshape(T, k), idx_ref)


@pytest.mark.parametrize("T,E,k,mode", [(1, 8, 2, "rand"), (33, 8, 2, "rand"), (4096, 8, 2, "rand"),
                                        (100, 8, 2, "one"), (64, 64, 8, "rand"), (0, 8, 2, "rand"),
                                        (17, 8, 2, "skip")])
def test_permute_bitexact(moe, orc, torch_mod, cuda, T, E, k, mode):
    torch = torch_mod
    rng = np.random.default_rng(T * 31 + E)
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32) if T else np.zeros((0, k), np.int32)
    if mode == "one":
        idx[:, 0] = 3
        idx[:, 1] = 6
    if mode == "skip":  # experts 0..3 never chosen
        idx = np.stack([rng.permutation(np.arange(4, E))[:k] for _ in range(T)]).astype(np.int32)
    ref = orc.permute(idx, T, E, k)
    n = max(T * k, 1)
    d_idx = to_dev(idx.reshape(-1) if T else np.zeros(1, np.int32), torch, cuda)
    counts = torch.full((E,), -1, dtype=torch.int32, device=cuda)
    offsets = torch.full((E + 1,), -1, dtype=torch.int32, device=cuda)
    perm = torch.full((n,), -1, dtype=torch.int32, device=cuda)
    inv = torch.full((n,), -1, dtype=torch.int32, device=cuda)
    moe.permute(d_idx, T, E, k, counts, offsets, perm, inv)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(counts, np.int32), ref[0])
    assert np.array_equal(to_np(offsets, np.int32), ref[1])
    if T:
        assert np.array_equal(to_np(perm, np.int32)[:T * k], ref[2])
        assert np.array_equal(to_np(inv, np.int32)[:T * k], ref[3])


def _expert_tensors(orc, torch, cuda, m, e, precision):
    """Host (logical) tensors for the oracle, device tensors in block layout."""
    d, f = m.d_model, m.d_ffn
    if precision == 1:
        gu, dn = orc.expert_bf16(m, e)
        dev = (to_dev(orc.pack_bf16_blocks(gu, 2 * f, d), torch, cuda), to_dev(orc.pack_bf16_blocks(dn, d, f), torch, cuda))
        return dev, (gu, dn)
    qgu, sgu, qd, sd = orc.expert_int4(m, e)
    qgub, sgub = orc.pack_int4_blocks(qgu, sgu, 2 * f, d)
    qdb, sdb = orc.pack_int4_blocks(qd, sd, d, f)
    dev = tuple(to_dev(a, torch, cuda) for a in (qgub, sgub, qdb, sdb))
    return dev, (qgu, sgu, qd, sd)


@pytest.mark.parametrize("T", [1, 2, 3, 4, 6, 8, 13])
@pytest.mark.parametrize("mix", ["bf16", "int4", "mixed"])
@pytest.mark.parametrize("shape", [(512, 1792), (1024, 2048)])
def test_ffn_grouped_vs_oracle(moe, orc, torch_mod, cuda, T, mix, shape):
    torch = torch_mod
    (d, f), E, k = shape, 8, 2
    m = orc.model(1, E, k, d, f, 1234)
    prec = {"bf16": [1] * E, "int4": [0] * E, "mixed": [0, 1] * (E // 2)}[mix]
    x = orc.step_input(m, T, T)
    wg = orc.router_weights(m, 0)
    idx, w, _ = orc.gate_topk(x, wg, T, d, E, k)
    counts, offsets, perm, inv = orc.permute(idx, T, E, k)
    experts, host = [], {}
    keep = []
    for e in range(E):
        dev, h = _expert_tensors(orc, torch, cuda, m, e, prec[e])
        keep.append(dev)
        host[e] = h
        if prec[e] == 1:
            experts.append(moe.expert_weights(moe.MOE_P16, dev[0], dev[1]))
        else:
            experts.append(moe.expert_weights(moe.MOE_P4, dev[0], dev[2], dev[1], dev[3]))
    nws = moe.ffn_workspace_bytes(T, k, E, d, f)
    ws = torch.zeros(nws, dtype=torch.uint8, device=cuda)
    y = torch.full((T * k * d,), float("nan"), dtype=torch.float32, device=cuda)
    for _ in range(2):  # the workspace is reusable: counters return to zero
        moe.ffn(to_dev(x, torch, cuda), to_dev(perm, torch, cuda), to_dev(offsets, torch, cuda), T, k, experts, d,
                f, ws, nws, y)
    torch.cuda.synchronize()
    y = to_np(y, np.float32).reshape(T * k, d)
    for e in range(E):
        lo, hi = offsets[e], offsets[e + 1]
        if lo == hi:
            continue
        xs = x[perm[lo:hi] // k]
        if prec[e] == 1:
            y_ref = orc.ffn_bf16(xs, hi - lo, host[e][0], host[e][1], d, f)
        else:
            y_ref = orc.ffn_int4(xs, hi - lo, *host[e], d, f)
        assert_close(y[lo:hi], y_ref, RTOL_F32, f"expert {e} ({'bf16' if prec[e] else 'int4'})")


def _sample_rows(lo, hi, full):
    """All rows of a segment, or (large Mixtral segments) rows on both sides
    of every 128-token tile boundary plus the segment's last rows."""
    if full:
        return np.arange(lo, hi)
    picks = set()
    for b in range(0, hi - lo, 128):
        picks.update(lo + v for v in (b, b + 1, b + 127) if lo + v < hi)
    picks.update(range(max(lo, hi - 3), hi))
    return np.array(sorted(picks))


# T * k >= 128 * (active experts) selects the 256-token tile variant
# (tc_gemm.cu moek_ffn_tc): T = 520 / 777 (tiny, 8 active experts; 777 ends
# on a partial 256-token tile), skew (2 active experts, 600 slots), T = 1024
# at Mixtral shape; f = 1920 (odd row-tile count) for the non-pair fallback.
@pytest.mark.parametrize("mix", ["bf16", "int4", "mixed"])
@pytest.mark.parametrize("T,shape,skew", [(40, (512, 1792), False), (300, (512, 1792), False),
                                          (96, (4096, 14336), False), (520, (512, 1792), False),
                                          (777, (512, 1792), False), (300, (512, 1792), True),
                                          (1024, (4096, 14336), False), (520, (512, 1920), False)])
def test_ffn_tcgen05_vs_oracle(moe, orc, torch_mod, cuda, T, shape, skew, mix):
    """K3/K4 on tcgen05 (batched / prefill path): every expert's y rows vs
    the oracle FFN on the same tokens (bf16: BF16 operands; int4: on-chip
    fp16 q*s, exact dequant values).  Covers the 128- and 256-token tile
    variants, partial last tiles and skewed routing."""
    torch = torch_mod
    (d, f), E, k = shape, 8, 2
    m = orc.model(1, E, k, d, f, 99)
    prec = {"bf16": [1] * E, "int4": [0] * E, "mixed": [0, 1] * (E // 2)}[mix]
    x = orc.step_input(m, T, T)
    wg = orc.router_weights(m, 0)
    idx, w, _ = orc.gate_topk(x, wg, T, d, E, k)
    if skew:  # every token on experts 5 and 2 (one int4, one bf16 in the mixed plan)
        idx = np.tile(np.array([5, 2], np.int32), (T, 1))
    counts, offsets, perm, inv = orc.permute(idx, T, E, k)
    wide = T * k >= 128 * int((counts > 0).sum())
    assert wide == (T in (520, 777, 1024) or skew)
    # f = 1920: an odd count of 128-row tiles, so wide launches take the single-CTA
    # tc_ffn_wide (bf16) + tc_ffn_kernel<256> (int4) instead of the CTA-pair kernel
    experts, host, keep = [], {}, []
    for e in range(E):
        dev, h = _expert_tensors(orc, torch, cuda, m, e, prec[e])
        keep.append(dev)
        host[e] = h
        if prec[e] == 1:
            experts.append(moe.expert_weights(moe.MOE_P16, dev[0], dev[1]))
        else:
            experts.append(moe.expert_weights(moe.MOE_P4, dev[0], dev[2], dev[1], dev[3]))
    nws = moe.ffn_tc_workspace_bytes(T, k, d, f)
    ws = torch.empty(nws, dtype=torch.uint8, device=cuda)
    y = torch.full((T * k * d,), float("nan"), dtype=torch.float32, device=cuda)
    moe.ffn_tc(to_dev(x, torch, cuda), to_dev(perm, torch, cuda), to_dev(offsets, torch, cuda), T, k, experts, d, f,
               ws, nws, y)
    torch.cuda.synchronize()
    y = to_np(y, np.float32).reshape(T * k, d)
    assert np.isfinite(y).all(), "every slot is written"
    for e in range(E):
        lo, hi = offsets[e], offsets[e + 1]
        if lo == hi:
            continue
        rows = _sample_rows(lo, hi, full=d < 4096 or hi - lo <= 64)
        xs = x[perm[rows] // k]
        if prec[e] == 1:
            y_ref = orc.ffn_bf16(xs, len(rows), host[e][0], host[e][1], d, f)
        else:
            y_ref = orc.ffn_int4(xs, len(rows), *host[e], d, f)
        assert_close(y[rows], y_ref, RTOL_F32, f"expert {e} ({'bf16' if prec[e] else 'int4'})")


def test_combine_bitexact(moe, orc, torch_mod, cuda):
    torch = torch_mod
    T, d, k = 9, 512, 2
    rng = np.random.default_rng(5)
    y = rng.standard_normal((T * k, d)).astype(np.float32)
    inv = rng.permutation(T * k).astype(np.int32)
    w = rng.random((T, k)).astype(np.float32)
    res = orc.synth_input(1, 2, T * d)
    ref = orc.combine(y, inv, w, res, T, d, k)
    out = torch.empty(T * d, dtype=torch.int16, device=cuda)
    moe.combine(to_dev(y, torch, cuda), to_dev(inv, torch, cuda), to_dev(w, torch, cuda), to_dev(res, torch, cuda),
                T, d, k, out)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(out, np.uint16).reshape(T, d), ref)
    ref0 = orc.combine(y, inv, w, None, T, d, k)
    moe.combine(to_dev(y, torch, cuda), to_dev(inv, torch, cuda), to_dev(w, torch, cuda), None, T, d, k, out)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(out, np.uint16).reshape(T, d), ref0)


def test_no_fallback_errors_are_loud(moe, torch_mod, cuda):
    with pytest.raises(moe.UsageError):
        moe.gate_topk(None, None, 1, 100, 8, 2, None, None)  # d % 8 != 0
    with pytest.raises(moe.UsageError):
        moe.ffn(None, None, None, 1, 2, [], 512, 1792, None, 0, None)  # E = 0


def test_zero_tokens_are_noops(moe, orc, torch_mod, cuda):
    """T = 0 (an empty batch, or a rank whose shard got no slots) is valid
    input for every stateless entry point: nothing launches, nothing is
    written, and the call succeeds."""
    torch = torch_mod
    d, f, E, k = 512, 1792, 8, 2
    x = torch.zeros(d, dtype=torch.int16, device=cuda)
    wg = torch.zeros(E * d, dtype=torch.int16, device=cuda)
    idx = torch.full((k,), -7, dtype=torch.int32, device=cuda)
    w = torch.full((k,), -7.0, dtype=torch.float32, device=cuda)
    moe.gate_topk(x, wg, 0, d, E, k, idx, w)
    moe.route(x, wg, 0, d, E, k, 1e-5, idx, w)
    y = torch.full((k * d,), -7.0, dtype=torch.float32, device=cuda)
    m = orc.model(1, E, k, d, f, 5)
    dev, _ = _expert_tensors(orc, torch, cuda, m, 0, 1)
    experts = [moe.expert_weights(moe.MOE_P16, dev[0], dev[1])] * E
    offs = torch.zeros(E + 1, dtype=torch.int32, device=cuda)
    moe.ffn(x, idx, offs, 0, k, experts, d, f, None, 0, y)
    moe.ffn_tc(x, idx, offs, 0, k, experts, d, f, None, 0, y)
    out = torch.full((d,), -7, dtype=torch.int16, device=cuda)
    moe.combine(y, idx, w, None, 0, d, k, out)
    torch.cuda.synchronize()
    assert (idx == -7).all() and (w == -7.0).all() and (y == -7.0).all() and (out == -7).all()
