"""The fused batch-1 decode step (gemv.cu decode_step_kernel: the whole stack
in one cooperative launch, grid barriers between phases) against the
per-layer kernels: outputs and routing bit-identical step after step, graph
and eager, tiny and Mixtral shapes, every precision mix."""
import numpy as np
import pytest

from helpers import MIXTRAL, TINY, read_device

pytestmark = pytest.mark.gpu


def _pair(moe, cfg, n4, seed, eps, graphs=True, plan_seed=0):
    prof = moe.profile_for_shape(cfg["d_model"], cfg["d_ffn"], cfg["num_layers"], cfg["experts_per_layer"],
                                 cfg["top_k"])
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, plan_seed), moe.HardwareProfile(10**15), prof)
    mk = lambda per_layer: moe.MoeEngine(cfg["num_layers"], cfg["experts_per_layer"], cfg["top_k"], cfg["d_model"],
                                         cfg["d_ffn"], plan, max_tokens=1, seed=seed, norm_eps=eps,
                                         use_graphs=graphs, per_layer_decode=per_layer)
    return mk(False), mk(True)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("eps", [0.0, 1e-5])
@pytest.mark.parametrize("n4", [0, 8, 16])
def test_fused_equals_per_layer_tiny(moe, cuda, n4, eps, graphs):
    import torch
    fused, ref = _pair(moe, TINY, n4, 42, eps, graphs, plan_seed=1)
    assert fused.profile_fused() is not None and ref.profile_fused() is None
    for step in range(24):
        for e in (fused, ref):
            e.synth_input(step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, fused.output_ptr, 1024), read_device(torch, ref.output_ptr, 1024)), step
        assert fused.last_routing(1) == ref.last_routing(1), step
    c = fused.counters()
    assert c.tokens == 24 and c.activations == 24 * 2 * 2 == c.hits
    fused.close()
    ref.close()


@pytest.mark.parametrize("n4", [0, 128, 256])
def test_fused_equals_per_layer_mixtral(moe, cuda, n4):
    import torch
    fused, ref = _pair(moe, MIXTRAL, n4, 0, 1e-5)
    for step in range(6):
        for e in (fused, ref):
            e.synth_input(1000 + step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, fused.output_ptr, 8192), read_device(torch, ref.output_ptr, 8192)), step
        assert fused.last_routing(1) == ref.last_routing(1), step
    ms, nbytes = fused.profile_fused()
    assert ms > 0 and nbytes > 32 * 2 * moe.expert_size(moe.profile_for_shape(4096, 14336, 32), 0)
    fused.close()
    ref.close()


@pytest.mark.parametrize("shape,n4", [("tiny", 8), ("mixtral", 128), ("mixtral", 256)])
def test_flow_equals_step(moe, cuda, monkeypatch, shape, n4):
    """The dataflow step (decode_flow_kernel, counters) and the grid-barrier
    step (decode_step_kernel) give bit-identical outputs and routing."""
    import torch
    cfg = TINY if shape == "tiny" else MIXTRAL
    prof = moe.profile_for_shape(cfg["d_model"], cfg["d_ffn"], cfg["num_layers"], cfg["experts_per_layer"],
                                 cfg["top_k"])
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, 1), moe.HardwareProfile(10**15), prof)
    engs = []
    for mode in ("flow", "step"):
        monkeypatch.setenv("MOE_FUSED", mode)
        engs.append(moe.MoeEngine(cfg["num_layers"], cfg["experts_per_layer"], cfg["top_k"], cfg["d_model"],
                                  cfg["d_ffn"], plan, max_tokens=1, seed=3, norm_eps=1e-5))
    n = 2 * cfg["d_model"]
    for step in range(8):
        for e in engs:
            e.synth_input(500 + step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, engs[0].output_ptr, n), read_device(torch, engs[1].output_ptr, n)), step
        assert engs[0].last_routing(1) == engs[1].last_routing(1), step
    for e in engs:
        e.close()


@pytest.mark.parametrize("shape", [
    dict(num_layers=3, experts_per_layer=8, top_k=1, d_model=512, d_ffn=1792),     # one slot per token
    dict(num_layers=2, experts_per_layer=16, top_k=2, d_model=768, d_ffn=640),     # 5 h groups: one partial chunk
    dict(num_layers=2, experts_per_layer=4, top_k=2, d_model=1024, d_ffn=2176),    # 17 groups: 3 chunks, last of 1
])
def test_flow_odd_shapes_equal_per_layer(moe, cuda, shape):
    """decode_flow_kernel at shapes the Mixtral tests do not reach (k = 1, E = 16,
    h-chunk counts with a partial last chunk) against the per-layer kernels."""
    import torch
    prof = moe.profile_for_shape(shape["d_model"], shape["d_ffn"], shape["num_layers"], shape["experts_per_layer"],
                                 shape["top_k"])
    n_exp = shape["num_layers"] * shape["experts_per_layer"]
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, n_exp // 2, 5), moe.HardwareProfile(10**15), prof)
    mk = lambda per_layer: moe.MoeEngine(shape["num_layers"], shape["experts_per_layer"], shape["top_k"],
                                         shape["d_model"], shape["d_ffn"], plan, max_tokens=1, seed=11,
                                         norm_eps=1e-5, per_layer_decode=per_layer)
    fused, ref = mk(False), mk(True)
    assert fused.profile_fused() is not None
    n = 2 * shape["d_model"]
    for step in range(10):
        for e in (fused, ref):
            e.synth_input(77 + step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, fused.output_ptr, n), read_device(torch, ref.output_ptr, n)), step
        assert fused.last_routing(1) == ref.last_routing(1), step
    fused.close()
    ref.close()


@pytest.mark.parametrize("shape,n4,steps", [("tiny", 8, 150), ("mixtral", 128, 20), ("mixtral", 256, 20)])
def test_flow_back_to_back_launches(moe, cuda, shape, n4, steps):
    """Two dataflow launches queued back to back (no host sync between): the
    second starts on the row buffers and counters the first left behind
    (sentinel rows reset by its last CTA out), so every checked step also
    checks the previous launch's clean-up.  Bit-identical to the per-layer
    kernels on the same inputs."""
    import torch
    cfg = TINY if shape == "tiny" else MIXTRAL
    flow, ref = _pair(moe, cfg, n4, 7, 1e-5, plan_seed=2)
    assert flow.profile_fused() is not None
    n = 2 * cfg["d_model"]
    for step in range(steps):
        for e in (flow, ref):
            e.synth_input(900 + step, 1)
            e.decode(1)
            e.synth_input(3000 + step, 1)
            e.decode(1)
            e.sync()
        assert np.array_equal(read_device(torch, flow.output_ptr, n), read_device(torch, ref.output_ptr, n)), step
        assert flow.last_routing(1) == ref.last_routing(1), step
    flow.close()
    ref.close()
