"""Expert parallelism over the GPUs of one box.

The reference is single-GPU. This is the north
star's addition: the expert set of every layer shards across G ranks, and
tokens stay data-parallel.

- Slot s of every layer belongs to rank floor(s*G/E), so E=8 / G=8 gives one
  slot per rank per layer. Router weights and the non-expert parts are
  replicated.
- Each rank may plan its own 256/G experts with make_plan (the placement is
  per rank).

Per layer (one process per GPU, torch.distributed for the exchange):

  1. all-gather the token rows of every rank (T = G * T_local rows);
  2. every rank routes all T tokens with the replicated router (K1+K2 fused,
     moe_route), so the routing is bit-identical everywhere and no routing
     message is needed;
  3. every rank computes only its own experts (moe_ffn / moe_ffn_tc with the
     other shards' weights NULL);
  4. it forms its share of each token's gate-weighted sum (moe_combine_partial);
  5. a reduce-scatter hands each token's summed share back to its owner,
     which adds the residual: out = bf16(x + sum) (moe_residual_add).

At batch 1 per GPU the exchange is latency-bound. The messages are 2*d bytes
per token (all-gather) and 4*d bytes per token (reduce-scatter). That costs
less than the per-(token, expert) all-to-all until T_local*k > G.

The arithmetic is the C-ABI kernels; the exchange is torch.distributed (NCCL
on GPUs). `ExpertParallelDecoder` takes an `ops` object, so that the CPU tests
can drive the same orchestration with gloo and the oracle.
"""
from __future__ import annotations

from typing import List, Sequence


def owner_of(slot: int, experts_per_layer: int, world: int) -> int:
    """Rank that owns expert slot `slot` of every layer."""
    return slot * world // experts_per_layer


def local_slots(rank: int, experts_per_layer: int, world: int) -> List[int]:
    return [s for s in range(experts_per_layer) if owner_of(s, experts_per_layer, world) == rank]


def expert_mask(rank: int, experts_per_layer: int, world: int) -> int:
    m = 0
    for s in local_slots(rank, experts_per_layer, world):
        m |= 1 << s
    return m


def exchange_bytes(T_local: int, world: int, d: int) -> dict:
    """Bytes one rank moves per layer: all-gather in (bf16 rows) and
    reduce-scatter out (fp32 shares)."""
    T = T_local * world
    return {"all_gather": (T - T_local) * d * 2, "reduce_scatter": (T - T_local) * d * 4}


def all_gather_rows(dist, out, inp, group=None):
    """out[rank*n:(rank+1)*n] = inp of every rank (any backend)."""
    if dist.get_backend(group) == "nccl":
        # NCCL has no int16: the rows are bf16 bits, move them as bfloat16
        torch = __import__("torch")
        dist.all_gather_into_tensor(out.view(torch.bfloat16), inp.view(torch.bfloat16), group=group)
    else:
        # gloo has no 16-bit integer type: move the bf16 rows as int32 pairs
        src = inp.view(inp.dtype if inp.element_size() == 4 else __import__("torch").int32)
        dst = out.view(src.dtype)
        n = src.numel()
        parts = [dst[r * n:(r + 1) * n] for r in range(dist.get_world_size(group))]
        dist.all_gather(parts, src, group=group)


def reduce_scatter_rows(dist, out, inp, group=None):
    """out = sum over ranks of inp[rank*n:(rank+1)*n] (any backend; gloo has
    no reduce-scatter, so it is an all-reduce + slice there)."""
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, inp, group=group)
    else:
        tmp = inp.clone()
        dist.all_reduce(tmp, group=group)
        n = out.numel()
        r = dist.get_rank(group)
        out.copy_(tmp[r * n:(r + 1) * n])


class CapiExchange:
    """The exchange through the C ABI (moe_ep_dispatch / moe_ep_combine on
    an NCCL communicator of the library's own), instead of
    torch.distributed's collectives.  `dist` only carries the unique id."""

    def __init__(self, moe, dist, rank: int, world: int, device: int, stream_fn):
        obj = [moe.ep_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        self.comm = moe.EpComm(obj[0], world, rank, device)
        self.stream_fn = stream_fn

    def all_gather_rows(self, out, inp):
        n = inp.numel()
        self.comm.dispatch(inp, 1, n, out, self.stream_fn())

    def reduce_scatter_rows(self, out, inp):
        self.comm.combine(inp, 1, out.numel(), out, self.stream_fn())

    def close(self):
        self.comm.close()


class PeerExchange:
    """The exchange fused into kernels over peer memory (kernels/ep_peer.cu):
    rows are pushed straight into every peer's gather buffer, shares straight
    into their owner's receive buffer, each followed by a system-scope
    release flag; no collective.  Buffers are shared by CUDA IPC handles
    (one process per GPU), or passed in directly (`bases`: one process
    driving G virtual ranks, as the single-GPU tests do)."""

    fused = True

    def __init__(self, moe, torch, rank: int, world: int, T_local: int, d: int, device, dist=None, bases=None,
                 own=None):
        self.moe, self.torch, self.rank, self.world, self.T_local, self.d = moe, torch, rank, world, T_local, d
        self.nbytes = moe.ep_peer_bytes(world, T_local, d)
        self._alloc = None
        if bases is None:  # one process per GPU: own cudaMalloc allocation, IPC handles
            self._alloc = moe.ep_peer_alloc(self.nbytes)
            self.own_ptr = self._alloc
            h = moe.ep_peer_ipc_handle(self.own_ptr)
            handles = [None] * world
            dist.all_gather_object(handles, h)
            ptrs = [self.own_ptr if r == rank else moe.ep_peer_ipc_open(handles[r]) for r in range(world)]
        else:  # virtual ranks in one process: caller-owned zeroed buffers
            self.own_ptr = own.data_ptr()
            ptrs = bases
        self.bases = moe.PeerBases(ptrs)
        rows = T_local * world * d
        self.xg = torch.as_tensor(_DevView(self.own_ptr, rows), device=device)
        self.epoch = 0

    def push_rows(self, x_local, stream):
        self.epoch += 1
        self.moe.ep_push_rows(x_local, self.T_local, self.d, self.rank, self.bases, self.epoch, stream)

    def wait_rows(self, stream):
        self.moe.ep_wait_rows(self.own_ptr, self.world, self.T_local, self.d, self.epoch, stream)

    def push_shares(self, ops, y, mask, stream):
        self.moe.ep_push_shares(y, ops.inv, ops.w, ops.idx, mask, self.T_local, self.d, ops.k, self.rank, self.bases,
                                self.epoch, stream)

    def reduce(self, x_local, out_local, stream):
        self.moe.ep_reduce(x_local, self.T_local, self.d, self.rank, self.bases, self.epoch, out_local, stream)


class _DevView:
    """int16 view of a raw device allocation (the gather rows at the buffer's head)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False), "version": 3}


class ExpertParallelDecoder:
    """Decode through an L-layer MoE stack with the experts sharded across
    the ranks of `group`.  `ops` supplies the per-layer arithmetic:

      ops.route(layer, xg, T)              -> state (routing + normalised rows)
      ops.ffn(layer, state, T)             -> per-slot expert outputs of this rank's experts
      ops.combine_partial(state, y, mask, T, part)   part[T, d] fp32 share
      ops.residual_add(x_local, mine, out_local)     out = bf16(x + mine)
      ops.empty_rows(n, fp32) / ops.num_layers / ops.d
    """

    def __init__(self, dist, ops, rank: int, world: int, T_local: int, experts_per_layer: int, group=None,
                 exchange=None):
        self.dist, self.ops, self.rank, self.world, self.group = dist, ops, rank, world, group
        self.exchange = exchange  # CapiExchange, or None: torch.distributed collectives
        self.T_local, self.T = T_local, T_local * world
        self.mask = expert_mask(rank, experts_per_layer, world)
        d = ops.d
        self.xg = ops.empty_rows(self.T * d, False)
        self.part = ops.empty_rows(self.T * d, True)
        self.mine = ops.empty_rows(T_local * d, True)
        self.bufs = [ops.empty_rows(T_local * d, False), ops.empty_rows(T_local * d, False)]

    def layer(self, layer: int, x_local, out_local):
        ops, T = self.ops, self.T
        if getattr(self.exchange, "fused", False):
            ex, stream = self.exchange, ops._stream()
            ex.push_rows(x_local, stream)
            ex.wait_rows(stream)
            state = ops.route(layer, ex.xg, T)
            y = ops.ffn(layer, state, T)
            ex.push_shares(ops, y, self.mask, stream)
            ex.reduce(x_local, out_local, stream)
            return state
        if self.exchange is not None:
            self.exchange.all_gather_rows(self.xg, x_local)
        else:
            all_gather_rows(self.dist, self.xg, x_local, self.group)
        state = ops.route(layer, self.xg, T)
        y = ops.ffn(layer, state, T)
        ops.combine_partial(state, y, self.mask, T, self.part)
        if self.exchange is not None:
            self.exchange.reduce_scatter_rows(self.mine, self.part)
        else:
            reduce_scatter_rows(self.dist, self.mine, self.part, self.group)
        ops.residual_add(x_local, self.mine, out_local)
        return state

    def decode(self, x_local, layers: Sequence[int] = None):
        layers = range(self.ops.num_layers) if layers is None else layers
        src = x_local
        for i, l in enumerate(layers):
            dst = self.bufs[i & 1]
            self.layer(l, src, dst)
            src = dst
        return src


class EngineOps:
    """GPU arithmetic for ExpertParallelDecoder: the C-ABI kernels over a
    MoeEngine's weights (router of every layer, this rank's experts)."""

    def __init__(self, moe, torch, engine, rank: int, world: int, T: int, norm_eps: float, device,
                 tc_min_tokens: int = 32):
        self.moe, self.torch, self.eng = moe, torch, engine
        self.num_layers, self.E, self.k, self.d, self.f = engine.L, engine.E, engine.k, engine.d, engine.f
        self.norm_eps, self.device, self.T = norm_eps, device, T
        self.tc = T >= tc_min_tokens
        i32, f32 = torch.int32, torch.float32
        self.idx = torch.empty(T * self.k, dtype=i32, device=device)
        self.w = torch.empty(T * self.k, dtype=f32, device=device)
        self.counts = torch.empty(self.E, dtype=i32, device=device)
        self.offsets = torch.empty(self.E + 1, dtype=i32, device=device)
        self.perm = torch.empty(T * self.k, dtype=i32, device=device)
        self.inv = torch.empty(T * self.k, dtype=i32, device=device)
        self.ticket = torch.zeros(4, dtype=torch.uint8, device=device)
        self.xn = torch.empty(T * self.d, dtype=torch.int16, device=device)
        self.y = torch.empty(T * self.k * self.d, dtype=f32, device=device)
        if self.tc:
            self.nws = moe.ffn_tc_workspace_bytes(T, self.k, self.d, self.f)
        else:
            self.nws = moe.ffn_workspace_bytes(T, self.k, self.E, self.d, self.f)
        self.ws = torch.zeros(self.nws, dtype=torch.uint8, device=device)
        mine = set(local_slots(rank, self.E, world))
        self.experts = []
        for l in range(self.num_layers):
            row = []
            for s in range(self.E):
                ex, _loc = engine.expert(l, s)
                if s not in mine:
                    ex = moe.ExpertWeightsC(ex.precision, 0, None, None, None, None)
                row.append(ex)
            self.experts.append(row)

    def _stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def empty_rows(self, n: int, fp32: bool):
        return self.torch.zeros(n, dtype=self.torch.float32 if fp32 else self.torch.int16, device=self.device)

    def route(self, layer, xg, T):
        self.moe.route(xg, self.eng.router(layer), T, self.d, self.E, self.k, self.norm_eps, self.idx, self.w, None,
                       self.counts, self.offsets, self.perm, self.inv, self.xn, self.ticket, self._stream())
        return layer

    def ffn(self, layer, state, T):
        fn = self.moe.ffn_tc if self.tc else self.moe.ffn
        fn(self.xn, self.perm, self.offsets, T, self.k, self.experts[layer], self.d, self.f, self.ws, self.nws, self.y,
           self._stream())
        return self.y

    def combine_partial(self, state, y, mask, T, part):
        self.moe.combine_partial(y, self.inv, self.w, self.idx, mask, T, self.d, self.k, part, self._stream())

    def residual_add(self, x_local, mine, out_local):
        self.moe.residual_add(x_local, mine, x_local.numel(), out_local, self._stream())


class RoutedA2ADecoder:
    """Host mirror of the sharded engine's expert-parallel step
    (MoeEngine with ep_world > 1, kernels/ep_a2a.cu), over torch.distributed
    point-to-point messages, for the CPU (gloo) protocol tests.  Per layer:

      1. each rank routes its own T tokens (ops.route: RMSNorm + top-k);
      2. dispatch: entry e = t*k + j goes to the owner of expert idx[e]; every
         rank sends each peer a fixed C = T*k entry buffer of rows + meta
         (meta[e] = expert if that peer owns it, else -1 -- the engine writes
         the same meta, and only the routed rows);
      3. each owner runs its experts on the entries it received (ops.expert);
      4. return: the output row of entry e goes back to its source at e;
      5. combine: out[t] = bf16(x[t] + sum_j w[t,j] * y[t*k+j]) in j order.

    `ops`: route(layer, x_local[T*d] uint16) -> (idx[T*k], w[T*k], xn[T][d]);
    expert(layer, slot, rows[n][d]) -> y[n][d] fp32; combine(x_local, w, y, T)
    -> out[T*d] uint16; num_layers, d, k, E."""

    def __init__(self, dist, ops, rank: int, world: int, T_local: int):
        self.dist, self.ops, self.rank, self.world, self.T = dist, ops, rank, world, T_local
        self.E, self.k, self.d = ops.E, ops.k, ops.d
        self.C = T_local * ops.k
        self.mine = local_slots(rank, ops.E, world)

    def _exchange(self, send):
        """send[p] (one array per peer, equal shapes) -> recv[src]."""
        torch = __import__("torch")
        recv = [None] * self.world
        reqs = []
        for p in range(self.world):
            if p == self.rank:
                recv[p] = send[p].copy()
                continue
            buf = __import__("numpy").empty_like(send[p])
            recv[p] = buf
            reqs.append(self.dist.isend(torch.from_numpy(send[p]), p))
            reqs.append(self.dist.irecv(torch.from_numpy(buf), p))
        for r in reqs:
            r.wait()
        return recv

    def layer(self, layer: int, x_local):
        np = __import__("numpy")
        ops, E, k, d, C, G = self.ops, self.E, self.k, self.d, self.C, self.world
        idx, w, xn = ops.route(layer, x_local)
        owner = [owner_of(int(s), E, G) for s in idx]
        rows = [np.zeros((C, d), np.uint16) for _ in range(G)]
        meta = [np.full(C, -1, np.int32) for _ in range(G)]
        for e in range(C):
            rows[owner[e]][e] = xn[e // k]
            meta[owner[e]][e] = idx[e]
        rrows, rmeta = self._exchange(rows), self._exchange(meta)
        ret = [np.zeros((C, d), np.float32) for _ in range(G)]
        for s in self.mine:  # this rank's experts on what it received, in (src, entry) order
            at = [(src, e) for src in range(G) for e in range(C) if rmeta[src][e] == s]
            if not at:
                continue
            y = ops.expert(layer, s, np.stack([rrows[src][e] for src, e in at]))
            for (src, e), yr in zip(at, y):
                ret[src][e] = yr
        back = self._exchange(ret)
        y_local = np.stack([back[owner[e]][e] for e in range(C)])
        return ops.combine(x_local, w, y_local, self.T)

    def decode(self, x_local, layers: Sequence[int] = None):
        layers = range(self.ops.num_layers) if layers is None else layers
        for l in layers:
            x_local = self.layer(l, x_local)
        return x_local
