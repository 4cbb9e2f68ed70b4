"""Expert parallelism.

CPU: two gloo ranks run the ExpertParallelDecoder orchestration (all-gather
of the rows, replicated routing, own-expert FFN, partial combine,
reduce-scatter, residual). The per-rank arithmetic is the CPU oracle
(test-only). The test checks the result against the single-process oracle
stack.

GPU: G virtual ranks in one process use the real kernels (moe_route, the
masked moe_ffn / moe_ffn_tc, moe_combine_partial, moe_residual_add). Their
summed shares must reproduce the engine's layer output.
"""
import os
import socket

import numpy as np
import pytest

from helpers import RTOL_BF16, TINY, assert_close, bf16_to_f32, to_dev, to_np

E, K, D, F, L, SEED, EPS = 8, 2, 512, 1792, 2, 77, 1e-5


def _bf16_rne(x):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


class OracleOps:
    """Per-rank arithmetic of the EP decoder on the CPU oracle (test-only)."""

    def __init__(self, torch, orc, m, precisions, rank, world):
        from paper_2407_14417_b200 import ep
        self.torch, self.orc, self.m = torch, orc, m
        self.num_layers, self.d = m.num_layers, m.d_model
        self.prec = precisions
        self.mine = set(ep.local_slots(rank, m.num_experts, world))
        self.wg = [orc.router_weights(m, l) for l in range(m.num_layers)]
        self.ex = {}
        for l in range(m.num_layers):
            for s in self.mine:
                e = l * m.num_experts + s
                self.ex[(l, s)] = orc.expert_bf16(m, e) if precisions[e] == 1 else orc.expert_int4(m, e)

    def empty_rows(self, n, fp32):
        return self.torch.zeros(n, dtype=self.torch.float32 if fp32 else self.torch.int16)

    def route(self, layer, xg, T):
        m, orc = self.m, self.orc
        x = xg.numpy().view(np.uint16).reshape(T, self.d)
        xn = orc.rmsnorm(x, T, self.d, m.norm_eps)
        idx, w, _ = orc.gate_topk(xn, self.wg[layer], T, self.d, m.num_experts, m.top_k)
        counts, offsets, perm, inv = orc.permute(idx, T, m.num_experts, m.top_k)
        return dict(layer=layer, xn=xn, idx=idx.reshape(-1), w=w.reshape(-1), offsets=offsets, perm=perm, inv=inv)

    def ffn(self, layer, st, T):
        m, orc, k = self.m, self.orc, self.m.top_k
        y = np.zeros((T * k, self.d), np.float32)
        for s in self.mine:
            lo, hi = st["offsets"][s], st["offsets"][s + 1]
            if lo == hi:
                continue
            xs = st["xn"][st["perm"][lo:hi] // k]
            w = self.ex[(layer, s)]
            if self.prec[layer * m.num_experts + s] == 1:
                y[lo:hi] = orc.ffn_bf16(xs, hi - lo, w[0], w[1], self.d, m.d_ffn)
            else:
                y[lo:hi] = orc.ffn_int4(xs, hi - lo, *w, self.d, m.d_ffn)
        return y

    def combine_partial(self, st, y, mask, T, part):
        k = self.m.top_k
        out = np.zeros((T, self.d), np.float32)
        for t in range(T):
            for j in range(k):
                if (mask >> int(st["idx"][t * k + j])) & 1:
                    out[t] = (np.float64(st["w"][t * k + j]) * y[st["inv"][t * k + j]] + out[t]).astype(np.float32)
        part.copy_(self.torch.from_numpy(out.reshape(-1)))

    def residual_add(self, x_local, mine, out_local):
        x = bf16_to_f32(x_local.numpy().view(np.uint16))
        out_local.copy_(self.torch.from_numpy(_bf16_rne(x + mine.numpy()).view(np.int16)))


def _ep_worker(rank, world, port, T_local, q):
    import torch
    import torch.distributed as dist

    from oracle.oracle import OracleLib
    from paper_2407_14417_b200 import ep
    import paper_2407_14417_b200 as moe
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = None
    try:
        orc = OracleLib()
        m = orc.model(L, E, K, D, F, SEED, EPS)
        prof = moe.profile_for_shape(D, F, L)
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
        ops = OracleOps(torch, orc, m, plan.precision, rank, world)
        dec = ep.ExpertParallelDecoder(dist, ops, rank, world, T_local, E)
        T = T_local * world
        x_all = orc.step_input(m, 5, T)
        x_local = torch.from_numpy(x_all[rank * T_local:(rank + 1) * T_local].reshape(-1).view(np.int16).copy())
        out = dec.decode(x_local).numpy().view(np.uint16).copy()
    except Exception as exc:  # report instead of leaving the peer waiting
        out = repr(exc)
    finally:
        q.put((rank, out))
        dist.destroy_process_group()


class OracleA2AOps:
    """Per-rank arithmetic of the routed all-to-all mirror (ep.RoutedA2ADecoder)
    on the CPU oracle (test-only): this rank's experts only."""

    def __init__(self, orc, m, precisions, rank, world):
        from paper_2407_14417_b200 import ep
        self.orc, self.m, self.prec = orc, m, precisions
        self.num_layers, self.d, self.k, self.E = m.num_layers, m.d_model, m.top_k, m.num_experts
        self.wg = [orc.router_weights(m, l) for l in range(m.num_layers)]
        self.ex = {}
        for l in range(m.num_layers):
            for s in ep.local_slots(rank, m.num_experts, world):
                e = l * m.num_experts + s
                self.ex[(l, s)] = orc.expert_bf16(m, e) if precisions[e] == 1 else orc.expert_int4(m, e)

    def route(self, layer, x_local):
        T = x_local.size // self.d
        xn = self.orc.rmsnorm(x_local.reshape(T, self.d), T, self.d, self.m.norm_eps)
        idx, w, _ = self.orc.gate_topk(xn, self.wg[layer], T, self.d, self.E, self.k)
        return idx.reshape(-1), w.reshape(-1), xn

    def expert(self, layer, s, rows):
        w = self.ex[(layer, s)]
        if self.prec[layer * self.E + s] == 1:
            return self.orc.ffn_bf16(rows, len(rows), w[0], w[1], self.d, self.m.d_ffn)
        return self.orc.ffn_int4(rows, len(rows), *w, self.d, self.m.d_ffn)

    def combine(self, x_local, w, y, T):
        inv = np.arange(T * self.k, dtype=np.int32)
        return self.orc.combine(np.ascontiguousarray(y, np.float32), inv, np.ascontiguousarray(w, np.float32),
                                x_local.reshape(T, self.d), T, self.d, self.k).reshape(-1)


def _a2a_worker(rank, world, port, T_local, q):
    import torch.distributed as dist

    from oracle.oracle import OracleLib
    from paper_2407_14417_b200 import ep
    import paper_2407_14417_b200 as moe
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = None
    try:
        orc = OracleLib()
        m = orc.model(L, E, K, D, F, SEED, EPS)
        prof = moe.profile_for_shape(D, F, L)
        plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
        dec = ep.RoutedA2ADecoder(dist, OracleA2AOps(orc, m, plan.precision, rank, world), rank, world, T_local)
        x_all = orc.step_input(m, 5, T_local * world)
        out = dec.decode(x_all[rank * T_local:(rank + 1) * T_local].reshape(-1).copy()).copy()
    except Exception as exc:  # report instead of leaving the peers waiting
        out = repr(exc)
    finally:
        q.put((rank, out))
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_and_exchange_sizes():
    from paper_2407_14417_b200 import ep
    assert [ep.owner_of(s, 8, 8) for s in range(8)] == list(range(8))
    assert [ep.owner_of(s, 8, 2) for s in range(8)] == [0, 0, 0, 0, 1, 1, 1, 1]
    assert ep.local_slots(1, 8, 4) == [2, 3]
    masks = [ep.expert_mask(r, 8, 4) for r in range(4)]
    assert sum(masks) == 0xFF and all(a & b == 0 for i, a in enumerate(masks) for b in masks[i + 1:])
    assert ep.exchange_bytes(1, 8, 4096) == {"all_gather": 7 * 8192, "reduce_scatter": 7 * 16384}


@pytest.mark.parametrize("T_local", [1, 3])
def test_ep_two_ranks_gloo_matches_single_process(orc, T_local):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, 2, port, T_local, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert not isinstance(res[r], str), f"rank {r}: {res[r]}"
    for p in procs:
        assert p.exitcode == 0
    import paper_2407_14417_b200 as moe
    m = orc.model(L, E, K, D, F, SEED, EPS)
    prof = moe.profile_for_shape(D, F, L)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    T = 2 * T_local
    x = orc.step_input(m, 5, T)
    for l in range(L):
        x, _, _, _ = orc.moe_layer(m, l, plan.precision[l * E:(l + 1) * E], x, T)
    got = np.concatenate([res[0].reshape(T_local, D), res[1].reshape(T_local, D)])
    assert_close(bf16_to_f32(got), bf16_to_f32(x), RTOL_BF16, "EP(2 ranks) vs single process")


@pytest.mark.gpu
@pytest.mark.parametrize("world,T", [(2, 3), (4, 4), (8, 8), (2, 96)])
def test_ep_virtual_ranks_gpu(moe, cuda, world, T):
    """The EP kernels on one GPU: G virtual ranks' shares summed == engine."""
    import torch
    from paper_2407_14417_b200 import ep
    prof = moe.profile_for_shape(D, F, L)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(L, E, K, D, F, plan, max_tokens=T, seed=SEED, use_graphs=False, norm_eps=EPS,
                        tc_min_tokens=64)
    eng.synth_input(2, T)
    eng.sync()
    x = torch.empty(T * D, dtype=torch.int16, device=cuda)
    x.copy_(torch.as_tensor(_Dev(eng.input_ptr, T * D), device=cuda))
    ref = torch.empty_like(x)
    ridx = torch.empty(T * K, dtype=torch.int32, device=cuda)
    eng.forward_layer(0, x, T, ref, ridx)
    eng.sync()
    total = torch.zeros(T * D, dtype=torch.float32, device=cuda)
    for r in range(world):
        ops = ep.EngineOps(moe, torch, eng, r, world, T, EPS, cuda)
        ops.route(0, x, T)
        y = ops.ffn(0, 0, T)
        part = torch.zeros(T * D, dtype=torch.float32, device=cuda)
        ops.combine_partial(0, y, ep.expert_mask(r, E, world), T, part)
        total += part
        assert torch.equal(ops.idx, ridx)
    out = torch.empty_like(x)
    moe.residual_add(x, total, T * D, out)
    torch.cuda.synchronize()
    assert_close(bf16_to_f32(to_np(out, np.uint16)), bf16_to_f32(to_np(ref, np.uint16)), RTOL_BF16,
                 f"EP virtual ranks G={world}")
    eng.close()


class _Dev:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


def test_ep_capi_unique_id(moe):
    """moe_ep_unique_id needs NCCL but no GPU (bootstrap handle)."""
    uid = moe.ep_unique_id()
    assert len(uid) == 128 and any(uid)
    with pytest.raises(moe.MoeError):
        moe.EpComm(uid, 2, 5)  # rank outside the world: usage error before any NCCL call


@pytest.mark.gpu
@pytest.mark.parametrize("T_local", [1, 5])
def test_ep_capi_single_rank_gpu(moe, cuda, T_local):
    """World-1 C-ABI exchange: dispatch is a copy of the rows, combine a copy
    of the shares (the multi-rank semantics are NCCL's all-gather /
    reduce-scatter; one GPU per rank, so N > 1 runs under torchrun)."""
    import torch
    uid = moe.ep_unique_id()
    comm = moe.EpComm(uid, 1, 0, 0)
    x = torch.randint(-3000, 3000, (T_local * D,), dtype=torch.int16, device=cuda)
    xa = torch.zeros_like(x)
    comm.dispatch(x, T_local, D, xa, torch.cuda.current_stream().cuda_stream)
    p = torch.randn(T_local * D, device=cuda)
    m = torch.zeros_like(p)
    comm.combine(p, T_local, D, m, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(xa, x) and torch.equal(m, p)
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world,T_local", [(2, 2), (4, 1), (8, 1), (2, 48)])
def test_ep_peer_exchange_virtual_ranks_gpu(moe, cuda, world, T_local):
    """The fused peer-memory exchange (kernels/ep_peer.cu) with G virtual ranks
    in one process: phases in rank order on one stream (push rows -> route +
    own experts + push shares -> reduce), each rank's output rows equal to the
    engine's single-device layer."""
    import torch
    from paper_2407_14417_b200 import ep
    T = world * T_local
    prof = moe.profile_for_shape(D, F, L)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(L, E, K, D, F, plan, max_tokens=T, seed=SEED, use_graphs=False, norm_eps=EPS)
    eng.synth_input(3, T)
    eng.sync()
    x = torch.empty(T * D, dtype=torch.int16, device=cuda)
    x.copy_(torch.as_tensor(_Dev(eng.input_ptr, T * D), device=cuda))
    ref = torch.empty_like(x)
    eng.forward_layer(0, x, T, ref)
    eng.sync()
    nb = moe.ep_peer_bytes(world, T_local, D)
    bufs = [torch.zeros(nb, dtype=torch.uint8, device=cuda) for _ in range(world)]
    ptrs = [b.data_ptr() for b in bufs]
    ops = [ep.EngineOps(moe, torch, eng, r, world, T, EPS, cuda) for r in range(world)]
    exs = [ep.PeerExchange(moe, torch, r, world, T_local, D, cuda, bases=ptrs, own=bufs[r]) for r in range(world)]
    xl = [x[r * T_local * D:(r + 1) * T_local * D].clone() for r in range(world)]
    outs = [torch.empty_like(xl[r]) for r in range(world)]
    s = torch.cuda.current_stream().cuda_stream
    for step in range(2):  # two layer steps: epochs 1 and 2 reuse the buffers
        for r in range(world):
            exs[r].push_rows(xl[r], s)
        for r in range(world):
            exs[r].wait_rows(s)
            assert torch.equal(exs[r].xg[:T * D], x)
            ops[r].route(0, exs[r].xg, T)
            y = ops[r].ffn(0, 0, T)
            exs[r].push_shares(ops[r], y, ep.expert_mask(r, E, world), s)
        for r in range(world):
            exs[r].reduce(xl[r], outs[r], s)
        torch.cuda.synchronize()
        got = torch.cat(outs)
        assert_close(bf16_to_f32(to_np(got, np.uint16)), bf16_to_f32(to_np(ref, np.uint16)), RTOL_BF16,
                     f"EP peer exchange G={world} step {step}")
    eng.close()


@pytest.mark.gpu
def test_ep_peer_exchange_two_processes_ipc_gpu(cuda):
    """Two processes on one GPU share exchange buffers by CUDA IPC handles and
    run the fused path, phased and flags-only (tools/ep_ipc_check.py): each
    rank's rows equal the single-device layer."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                        os.path.join(root, "tools", "ep_ipc_check.py")], capture_output=True, text=True, timeout=240)
    lines = [l for l in r.stdout.splitlines() if l.startswith("rank") and "err" in l]
    assert r.returncode == 0 and len(lines) == 4, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("world,T_local", [(2, 1), (2, 3), (4, 2)])
def test_routed_a2a_gloo_matches_single_process(orc, world, T_local):
    """The sharded engine's protocol (routed rows to owners, outputs back,
    combine) with gloo ranks and the oracle as per-rank arithmetic equals the
    single-process oracle stack."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, T_local, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert not isinstance(res[r], str), f"rank {r}: {res[r]}"
    import paper_2407_14417_b200 as moe
    m = orc.model(L, E, K, D, F, SEED, EPS)
    prof = moe.profile_for_shape(D, F, L)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    T = world * T_local
    x = orc.step_input(m, 5, T)
    for l in range(L):
        x, _, _, _ = orc.moe_layer(m, l, plan.precision[l * E:(l + 1) * E], x, T)
    got = np.concatenate([res[r].reshape(T_local, D) for r in range(world)])
    # the same per-entry arithmetic as the single process: bit-identical
    assert np.array_equal(got, x.reshape(T, D)), "routed all-to-all (oracle arithmetic) differs from single process"
