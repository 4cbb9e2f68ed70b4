"""Cross-process check of the fused peer-memory EP exchange (CUDA IPC handles),
on ONE GPU: two processes share cuda:0, exchange IPC handles over gloo and run
the decoder's fused layer path; each compares its rows with the single-device
layer.  The two contexts time-slice, so the flag waits make progress but slowly.
usage: torchrun --standalone --nproc-per-node 2 tools/ep_ipc_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2407_14417_b200 as moe
from paper_2407_14417_b200 import ep

L, E, K, D, F, SEED, EPS = 2, 8, 2, 512, 1792, 77, 1e-5


class _Dev:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda:0")
    T_local = 2
    T = T_local * world
    prof = moe.profile_for_shape(D, F, L)
    plan = moe.make_plan(moe.TaskRequest(moe.QUALITY, 8, 1), moe.HardwareProfile(10**15), prof)
    eng = moe.MoeEngine(L, E, K, D, F, plan, max_tokens=T, seed=SEED, use_graphs=False, norm_eps=EPS)
    eng.synth_input(4, T)
    eng.sync()
    x = torch.empty(T * D, dtype=torch.int16, device=dev)
    x.copy_(torch.as_tensor(_Dev(eng.input_ptr, T * D), device=dev))
    ref = torch.empty_like(x)
    eng.forward_layer(0, x, T, ref)
    eng.sync()
    ops = ep.EngineOps(moe, torch, eng, rank, world, T, EPS, dev)
    print(f"rank {rank}: engine ready", flush=True)
    ex = ep.PeerExchange(moe, torch, rank, world, T_local, D, dev, dist=dist)
    print(f"rank {rank}: IPC buffers open", flush=True)
    xl = x[rank * T_local * D:(rank + 1) * T_local * D].clone()
    out = torch.empty_like(xl)
    s = ops._stream()
    ex.push_rows(xl, s)
    torch.cuda.synchronize()
    print(f"rank {rank}: rows pushed", flush=True)
    dist.barrier()
    ex.wait_rows(s)
    torch.cuda.synchronize()
    print(f"rank {rank}: rows arrived", flush=True)
    ops.route(0, ex.xg, T)
    y = ops.ffn(0, 0, T)
    ex.push_shares(ops, y, ep.expert_mask(rank, E, world), s)
    torch.cuda.synchronize()
    print(f"rank {rank}: shares pushed", flush=True)
    dist.barrier()
    ex.reduce(xl, out, s)
    torch.cuda.synchronize()
    want = ref[rank * T_local * D:(rank + 1) * T_local * D]

    def rel_err(o):
        a = (o.cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        b = (want.cpu().numpy().view(np.uint16).astype(np.uint32) << 16).view(np.float32)
        return float(np.max(np.abs(a - b)) / max(1e-6, float(np.max(np.abs(b)))))

    err = rel_err(out)
    print(f"rank {rank}: phased (barriers) max rel err {err:.2e}", flush=True)
    # the decoder's fused layer path, no host barriers: the flags alone order the ranks
    dec = ep.ExpertParallelDecoder(dist, ops, rank, world, T_local, E, exchange=ex)
    out2 = torch.empty_like(xl)
    dec.layer(0, xl, out2)
    torch.cuda.synchronize()
    err = max(err, rel_err(out2))
    print(f"rank {rank}: decoder layer (flags only) max rel err {rel_err(out2):.2e}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if err < 1e-2 else 1)


if __name__ == "__main__":
    main()
