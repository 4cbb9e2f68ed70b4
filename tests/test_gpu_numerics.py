"""fp16-operand range guard of the int4 paths.

Both int4 paths multiply against fp16 copies of the bf16 activations, and
tcgen05 dequantises to fp16 q*s.  Out-of-range values must fail loudly
(ValidationError at the engine's sync, moe_numerics_status bits), while the
in-range cases the guard leaves alone stay exact:
  - the decoder-layer RMSNorm (unit weight) bounds |x| by sqrt(d), so a raw
    input far above 65504 is served exactly once normalised;
  - the GEMV applies the scale in fp32 after an integer-exact dot, so tiny
    scales are exact there (tcgen05 flags them); what flags on the GEMV is
    the activation group they produce downstream (h below 2^-14 throughout).
"""
import numpy as np
import pytest

from helpers import RTOL_BF16, assert_close, bf16_to_f32, to_dev, to_np

pytestmark = pytest.mark.gpu

D, F, E, K = 512, 1792, 8, 2


def _f32_to_bf16(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _engine(moe, prec, eps, T=1):
    prof = moe.profile_for_shape(D, F, 1, E, K)
    plan = moe.assign_locations(prec, moe.HardwareProfile(10**15), prof)
    return moe.MoeEngine(1, E, K, D, F, plan, max_tokens=T, seed=3, norm_eps=eps), plan


def _big_input(orc, m, T):
    x = bf16_to_f32(orc.step_input(m, 0, T)).astype(np.float32)
    x[:, 7] = 70000.0  # one channel far above the fp16 range
    return _f32_to_bf16(x)


def test_activation_overflow_raises_without_norm(moe, orc, cuda):
    import torch
    moe.numerics_status(clear=True)
    eng, _ = _engine(moe, [0] * E, 0.0)
    m = orc.model(1, E, K, D, F, 3)
    x = _big_input(orc, m, 1)
    out = torch.empty(D, dtype=torch.int16, device=cuda)
    eng.forward_layer(0, to_dev(x, torch, cuda), 1, out)
    with pytest.raises(moe.ValidationError, match="fp16"):
        eng.sync()
    assert moe.numerics_status() == 0, "sync clears the word"
    eng.close()


def test_bf16_plan_ignores_fp16_copies(moe, orc, cuda):
    """A bf16-only plan never computes on the fp16 copies: no error, and the
    output matches the oracle."""
    import torch
    moe.numerics_status(clear=True)
    eng, _ = _engine(moe, [1] * E, 0.0)
    m = orc.model(1, E, K, D, F, 3)
    x = _big_input(orc, m, 1)
    out = torch.empty(D, dtype=torch.int16, device=cuda)
    eng.forward_layer(0, to_dev(x, torch, cuda), 1, out)
    eng.sync()
    ref, _, _, _ = orc.moe_layer(m, 0, [1] * E, x, 1)
    assert_close(bf16_to_f32(to_np(out, np.uint16)), bf16_to_f32(ref.reshape(-1)), RTOL_BF16, "bf16 plan")
    moe.numerics_status(clear=True)
    eng.close()


@pytest.mark.parametrize("T", [1, 40])
def test_rmsnorm_keeps_large_inputs_in_range(moe, orc, cuda, T):
    """|x| = 70000 on the raw residual: RMSNorm (unit weight) maps it below
    sqrt(d), the int4 paths (GEMV at T=1, tcgen05 at T=40) run in range and
    match the oracle."""
    import torch
    moe.numerics_status(clear=True)
    prof = moe.profile_for_shape(D, F, 1, E, K)
    plan = moe.assign_locations([0, 1] * (E // 2), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(1, E, K, D, F, plan, max_tokens=T, seed=3, norm_eps=1e-5, tc_min_tokens=16)
    m = orc.model(1, E, K, D, F, 3, 1e-5)
    x = _big_input(orc, m, T)
    out = torch.empty(T * D, dtype=torch.int16, device=cuda)
    eng.forward_layer(0, to_dev(x, torch, cuda), T, out)
    eng.sync()
    ref, _, _, _ = orc.moe_layer(m, 0, [0, 1] * (E // 2), x, T)
    assert_close(bf16_to_f32(to_np(out, np.uint16).reshape(T, D)), bf16_to_f32(ref), RTOL_BF16, "normed")
    eng.close()


def test_tiny_weights_flagged(moe, orc, cuda):
    """int4-g128 scales ~2^-27 (weights scaled by 2^-20): the GEMV's gate/up
    dot applies them in fp32, but the SwiGLU output h is ~1e-13, below the
    fp16 normal range in every group, so its fp16 copy would flush -- the
    GEMV raises the activation bit; tcgen05's fp16 q*s would be subnormal,
    so it raises the scale bit.  Neither returns silently wrong values."""
    import torch
    moe.numerics_status(clear=True)
    T = 3
    m = orc.model(1, E, K, D, F, 77)
    gu, dn = orc.expert_bf16(m, 0)
    tiny = [_f32_to_bf16(bf16_to_f32(a).astype(np.float32) * np.float32(2.0 ** -20)) for a in (gu, dn)]
    qgu, sgu = orc.quantize(tiny[0], 2 * F, D)
    qd, sd = orc.quantize(tiny[1], D, F)
    assert bf16_to_f32(sgu).max() < 2.0 ** -14
    qgub, sgub = orc.pack_int4_blocks(qgu, sgu, 2 * F, D)
    qdb, sdb = orc.pack_int4_blocks(qd, sd, D, F)
    dev = [to_dev(a, torch, cuda) for a in (qgub, sgub, qdb, sdb)]
    ex = moe.expert_weights(moe.MOE_P4, dev[0], dev[2], dev[1], dev[3])
    x = orc.step_input(m, 1, T)
    perm = np.arange(T * K, dtype=np.int32)
    offsets = np.array([0] + [T * K] * E, np.int32)  # every slot on expert 0
    y = torch.empty(T * K * D, dtype=torch.float32, device=cuda)
    nws = moe.ffn_workspace_bytes(T, K, E, D, F)
    ws = torch.zeros(nws, dtype=torch.uint8, device=cuda)
    moe.ffn(to_dev(x, torch, cuda), to_dev(perm, torch, cuda), to_dev(offsets, torch, cuda), T, K, [ex] * E, D, F,
            ws, nws, y)
    torch.cuda.synchronize()
    assert moe.numerics_status() == moe.NUMERICS_F16_ACTIVATION
    nws = moe.ffn_tc_workspace_bytes(T, K, D, F)
    wst = torch.empty(nws, dtype=torch.uint8, device=cuda)
    moe.ffn_tc(to_dev(x, torch, cuda), to_dev(perm, torch, cuda), to_dev(offsets, torch, cuda), T, K, [ex] * E, D, F,
               wst, nws, y)
    torch.cuda.synchronize()
    assert moe.numerics_status() & moe.NUMERICS_F16_SCALE


def test_normal_data_never_flags(moe, orc, cuda):
    """The guard has no false alarms on the synthetic Mixtral-style data:
    a mixed-precision tiny-shape stack decodes 16 steps on both paths with
    the word clear."""
    import torch  # noqa: F401
    moe.numerics_status(clear=True)
    prof = moe.profile_for_shape(D, F, 2, E, K)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    for T, tc in ((1, 0), (40, 16)):
        eng = moe.MoeEngine(2, E, K, D, F, plan, max_tokens=T, seed=5, norm_eps=1e-5, tc_min_tokens=tc)
        for step in range(16):
            eng.synth_input(step, T)
            eng.decode(T)
        eng.sync()  # raises on any flag
        eng.close()
    assert moe.numerics_status() == 0
