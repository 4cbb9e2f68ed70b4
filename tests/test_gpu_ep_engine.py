"""Sharded expert parallelism on one GPU with virtual ranks:
G MoeEngines with ep_world = G each hold only their own slots' experts and
exchange routed rows over peer memory (ep_a2a.cu) inside decode().  Checked
against one single-device engine holding every expert, on the same weights
and the same G*T tokens: routing of every layer bit-exact per token, layer
outputs within the bf16 tolerance (the owners run the GEMV / tcgen05 GEMM on
their received rows, so K-part decompositions -- and fp32 rounding -- may
differ from the single-device batch), and each rank's expert memory 1/G of
the whole.  Ranks decode concurrently (one host thread each: a rank's step
waits on its peers' flags)."""
import threading

import numpy as np
import pytest

from helpers import MIXTRAL, RTOL_BF16, TINY, assert_close, bf16_to_f32, read_device

pytestmark = pytest.mark.gpu


class _DevBytes:
    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}


def write_device(torch, ptr, data: np.ndarray):
    dst = torch.as_tensor(_DevBytes(ptr, data.nbytes), device="cuda")
    dst.copy_(torch.from_numpy(np.ascontiguousarray(data).reshape(-1).view(np.uint8)))
    torch.cuda.synchronize()


def quality_plan(moe, cfg, n4, seed):
    prof = moe.profile_for_shape(cfg["d_model"], cfg["d_ffn"], cfg["num_layers"], cfg["experts_per_layer"],
                                 cfg["top_k"])
    return moe.make_plan(moe.TaskRequest(moe.QUALITY, n4, seed), moe.HardwareProfile(10**15), prof)


def engine(moe, cfg, plan, T, seed, eps, rank=0, world=1, graphs=True, tc_min=0):
    return moe.MoeEngine(cfg["num_layers"], cfg["experts_per_layer"], cfg["top_k"], cfg["d_model"], cfg["d_ffn"],
                         plan, max_tokens=T, seed=seed, use_graphs=graphs, norm_eps=eps, tc_min_tokens=tc_min,
                         ep_rank=rank, ep_world=world)


def sharded(moe, cfg, plan, G, T, seed, eps, graphs=True, tc_min=0):
    engs = [engine(moe, cfg, plan, T, seed, eps, r, G, graphs, tc_min) for r in range(G)]
    bases = [e.ep_buffer()[0] for e in engs]
    for e in engs:
        e.ep_set_peers(bases)
    return engs


def decode_all(engs, T, steps=1):
    errs = []

    def go(e):
        try:
            for _ in range(steps):
                e.decode(T)
            e.sync()
        except Exception as ex:  # noqa: BLE001 -- reported below
            errs.append(ex)

    th = [threading.Thread(target=go, args=(e,)) for e in engs]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank did not finish its decode step"
    assert not errs, errs


def check_against_single(moe, torch, cfg, plan, G, T, seed=5, eps=1e-5, step=11, graphs=True, tc_min=0, steps=1):
    d, L, k = cfg["d_model"], cfg["num_layers"], cfg["top_k"]
    single = engine(moe, cfg, plan, G * T, seed, eps, graphs=graphs, tc_min=tc_min)
    single.synth_input(step, G * T)
    x = read_device(torch, single.input_ptr, G * T * d * 2).view(np.uint16).reshape(G * T, d)
    single.decode(G * T)
    single.sync()
    ref = read_device(torch, single.output_ptr, G * T * d * 2).view(np.uint16).reshape(G * T, d)
    ref_route = np.array(single.last_routing(G * T)).reshape(G * T, L, k)
    engs = sharded(moe, cfg, plan, G, T, seed, eps, graphs, tc_min)
    for r, e in enumerate(engs):
        write_device(torch, e.input_ptr, x[r * T:(r + 1) * T])
    decode_all(engs, T, steps)
    for r, e in enumerate(engs):
        got = read_device(torch, e.output_ptr, T * d * 2).view(np.uint16).reshape(T, d)
        route = np.array(e.last_routing(T)).reshape(T, L, k)
        assert np.array_equal(route, ref_route[r * T:(r + 1) * T]), f"rank {r}: routing differs from the single engine"
        assert_close(bf16_to_f32(got), bf16_to_f32(ref[r * T:(r + 1) * T]), RTOL_BF16, f"rank {r} of {G} output")
    single_bytes = single.memory()["expert_bytes"]
    per_rank = [e.memory()["expert_bytes"] for e in engs]
    assert sum(per_rank) == single_bytes, "the shards must partition the experts"
    for e in engs:
        e.close()
    single.close()
    return per_rank, single_bytes


@pytest.fixture(scope="module")
def torch_mod(cuda):
    import torch
    return torch


@pytest.mark.parametrize("G,T", [(2, 1), (2, 3), (4, 1), (8, 1), (8, 2)])
def test_ep_sharded_equals_single_tiny_gemv(moe, torch_mod, cuda, G, T):
    plan = quality_plan(moe, TINY, 8, 1)
    per_rank, total = check_against_single(moe, torch_mod, TINY, plan, G, T)
    assert max(per_rank) <= total // G + total // TINY["experts_per_layer"], "a rank holds more than its shard"


@pytest.mark.parametrize("G", [2, 4])
def test_ep_sharded_equals_single_tiny_tcgen05(moe, torch_mod, cuda, G):
    # local batch 32 >= tc_min_tokens: owners run the tcgen05 GEMM on their received rows
    plan = quality_plan(moe, TINY, 8, 1)
    check_against_single(moe, torch_mod, TINY, plan, G, 32)


def test_ep_eager_equals_graph_and_repeats(moe, torch_mod, cuda):
    # several steps back to back (epochs advance inside the captured graph)
    plan = quality_plan(moe, TINY, 8, 1)
    check_against_single(moe, torch_mod, TINY, plan, 2, 2, graphs=False)
    check_against_single(moe, torch_mod, TINY, plan, 2, 2, graphs=True, steps=3)


def test_ep_mixtral_shape_two_ranks(moe, torch_mod, cuda):
    # 2 of Mixtral's 32 layers, mixed int4/bf16 per the quality plan
    cfg = dict(MIXTRAL, num_layers=2)
    plan = quality_plan(moe, cfg, 8, 0)
    per_rank, total = check_against_single(moe, torch_mod, cfg, plan, 2, 1)
    assert all(b < total for b in per_rank)


def test_ep_set_peers_validation(moe, cuda):
    plan = quality_plan(moe, TINY, 8, 1)
    engs = [engine(moe, TINY, plan, 1, 5, 1e-5, r, 2) for r in range(2)]
    with pytest.raises(moe.UsageError):
        engs[0].decode(1)  # peers not set
    with pytest.raises(moe.UsageError):
        engs[0].ep_set_peers([engs[1].ep_buffer()[0], engs[0].ep_buffer()[0]])  # own base not at ep_rank
    one = engine(moe, TINY, plan, 1, 5, 1e-5)
    with pytest.raises(moe.UsageError):
        one.ep_set_peers([one.ep_buffer()[0]])
    for e in engs + [one]:
        e.close()
