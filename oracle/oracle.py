"""ctypes access to the test-only checkers (TEST INFRASTRUCTURE ONLY).

  OracleLib -> oracle/build/libmoe_oracle.so : CPU restatement of the MoE math
  RefLib    -> oracle/_ref/libmoeserve_ref.so: the unmodified reference library
                compiled from /root/reference/proj/src (+ ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libmoe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoeserve_ref.so")

P = C.POINTER
VP = C.c_void_p


def _np_ptr(a):
    return a.ctypes.data_as(VP) if a is not None else None


class OrcModel(C.Structure):
    _fields_ = [("num_layers", C.c_int), ("num_experts", C.c_int), ("top_k", C.c_int), ("d_model", C.c_int),
                ("d_ffn", C.c_int), ("seed", C.c_uint64), ("norm_eps", C.c_float), ("pad_", C.c_int)]


class OrcExpert(C.Structure):
    _fields_ = [("precision", C.c_int), ("w_gate_up", VP), ("s_gate_up", VP), ("w_down", VP), ("s_down", VP)]


class OracleLib:
    """CPU restatement of K1-K5 + generators (oracle/moe_oracle.h)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        L = C.CDLL(path)
        I, U64, I64 = C.c_int, C.c_uint64, C.c_int64
        sig = {
            "orc_rand64": (U64, [U64, U64, U64]),
            "orc_synth_weight_bf16": (None, [U64, U64, I64, I, VP]),
            "orc_synth_input_bf16": (None, [U64, U64, I64, VP]),
            "orc_weight_shift": (I, [I]),
            "orc_quantize_g128": (None, [VP, I, I, VP, VP]),
            "orc_dequant_g128": (None, [VP, VP, I, I, VP]),
            "orc_gate_topk": (None, [VP, VP, I, I, I, I, VP, VP, VP]),
            "orc_permute": (None, [VP, I, I, I, VP, VP, VP, VP]),
            "orc_ffn_bf16": (None, [VP, I, VP, VP, I, I, VP]),
            "orc_ffn_int4": (None, [VP, I, VP, VP, VP, VP, I, I, VP]),
            "orc_combine": (None, [VP, VP, VP, VP, I, I, I, VP]),
            "orc_expert_bf16": (None, [P(OrcModel), I, VP, VP]),
            "orc_expert_int4": (None, [P(OrcModel), I, VP, VP, VP, VP]),
            "orc_router_weights": (None, [P(OrcModel), I, VP]),
            "orc_step_input": (None, [P(OrcModel), I, I, VP]),
            "orc_moe_layer": (None, [P(OrcModel), I, VP, VP, I, VP, VP, VP, VP]),
            "orc_moe_layer_w": (None, [P(OrcModel), VP, P(OrcExpert), VP, I, VP, VP, VP, VP]),
            "orc_num_threads": (I, []),
            "orc_rmsnorm": (None, [VP, I, I, C.c_float, VP]),
            "orc_perm_k": (I, [I]),
            "orc_pack_bf16_blocks": (None, [VP, I, I, VP]),
            "orc_unpack_bf16_blocks": (None, [VP, I, I, VP]),
            "orc_pack_int4_blocks": (None, [VP, VP, I, I, VP, VP]),
            "orc_unpack_int4_blocks": (None, [VP, VP, I, I, VP, VP]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        self.L = L

    # generators -----------------------------------------------------------
    def synth_weight(self, seed, uid, n, shift):
        out = np.empty(n, np.uint16)
        self.L.orc_synth_weight_bf16(seed, uid, n, shift, _np_ptr(out))
        return out

    def synth_input(self, seed, uid, n):
        out = np.empty(n, np.uint16)
        self.L.orc_synth_input_bf16(seed, uid, n, _np_ptr(out))
        return out

    def weight_shift(self, K):
        return self.L.orc_weight_shift(K)

    def model(self, L, E, k, d, f, seed, norm_eps=0.0):
        return OrcModel(L, E, k, d, f, seed, norm_eps, 0)

    def rmsnorm(self, x, T, d, eps):
        out = np.empty(T * d, np.uint16)
        self.L.orc_rmsnorm(_np_ptr(np.ascontiguousarray(x)), T, d, C.c_float(eps), _np_ptr(out))
        return out.reshape(T, d)

    def expert_bf16(self, m, e):
        gu = np.empty(2 * m.d_ffn * m.d_model, np.uint16)
        dn = np.empty(m.d_model * m.d_ffn, np.uint16)
        self.L.orc_expert_bf16(C.byref(m), e, _np_ptr(gu), _np_ptr(dn))
        return gu.reshape(2 * m.d_ffn, m.d_model), dn.reshape(m.d_model, m.d_ffn)

    def expert_int4(self, m, e):
        d, f = m.d_model, m.d_ffn
        qgu = np.empty(2 * f * d // 8, np.uint32)
        sgu = np.empty(2 * f * d // 128, np.uint16)
        qd = np.empty(d * f // 8, np.uint32)
        sd = np.empty(d * f // 128, np.uint16)
        self.L.orc_expert_int4(C.byref(m), e, _np_ptr(qgu), _np_ptr(sgu), _np_ptr(qd), _np_ptr(sd))
        return (qgu.reshape(2 * f, d // 8), sgu.reshape(2 * f, d // 128), qd.reshape(d, f // 8),
                sd.reshape(d, f // 128))

    def router_weights(self, m, layer):
        wg = np.empty(m.num_experts * m.d_model, np.uint16)
        self.L.orc_router_weights(C.byref(m), layer, _np_ptr(wg))
        return wg.reshape(m.num_experts, m.d_model)

    def step_input(self, m, step, T):
        x = np.empty(T * m.d_model, np.uint16)
        self.L.orc_step_input(C.byref(m), step, T, _np_ptr(x))
        return x.reshape(T, m.d_model)

    # device storage layout ------------------------------------------------
    def pack_bf16_blocks(self, w, rows, cols):
        out = np.empty(rows * cols, np.uint16)
        self.L.orc_pack_bf16_blocks(_np_ptr(np.ascontiguousarray(w, np.uint16)), rows, cols, _np_ptr(out))
        return out

    def pack_int4_blocks(self, q, s, rows, cols):
        qb = np.empty(rows * cols // 8, np.uint32)
        sb = np.empty(rows * cols // 128, np.uint16)
        self.L.orc_pack_int4_blocks(_np_ptr(np.ascontiguousarray(q, np.uint32)), _np_ptr(np.ascontiguousarray(s, np.uint16)),
                                    rows, cols, _np_ptr(qb), _np_ptr(sb))
        return qb, sb

    def unpack_int4_blocks(self, qb, sb, rows, cols):
        q = np.empty(rows * cols // 8, np.uint32)
        s = np.empty(rows * cols // 128, np.uint16)
        self.L.orc_unpack_int4_blocks(_np_ptr(np.ascontiguousarray(qb, np.uint32)), _np_ptr(np.ascontiguousarray(sb, np.uint16)),
                                      rows, cols, _np_ptr(q), _np_ptr(s))
        return q.reshape(rows, cols // 8), s.reshape(rows, cols // 128)

    def perm_k(self, k):
        return self.L.orc_perm_k(k)

    # math -------------------------------------------------------------------
    def quantize(self, w, rows, cols):
        q = np.empty(rows * cols // 8, np.uint32)
        s = np.empty(rows * cols // 128, np.uint16)
        self.L.orc_quantize_g128(_np_ptr(np.ascontiguousarray(w, np.uint16)), rows, cols, _np_ptr(q), _np_ptr(s))
        return q.reshape(rows, cols // 8), s.reshape(rows, cols // 128)

    def dequant(self, q, s, rows, cols):
        out = np.empty(rows * cols, np.float32)
        self.L.orc_dequant_g128(_np_ptr(np.ascontiguousarray(q)), _np_ptr(np.ascontiguousarray(s)), rows, cols,
                                _np_ptr(out))
        return out.reshape(rows, cols)

    def gate_topk(self, x, wg, T, d, E, k):
        idx = np.empty(T * k, np.int32)
        w = np.empty(T * k, np.float32)
        lg = np.empty(T * E, np.float32)
        self.L.orc_gate_topk(_np_ptr(np.ascontiguousarray(x)), _np_ptr(np.ascontiguousarray(wg)), T, d, E, k,
                             _np_ptr(idx), _np_ptr(w), _np_ptr(lg))
        return idx.reshape(T, k), w.reshape(T, k), lg.reshape(T, E)

    def permute(self, idx, T, E, k):
        counts = np.empty(E, np.int32)
        offsets = np.empty(E + 1, np.int32)
        perm = np.empty(T * k, np.int32)
        inv = np.empty(T * k, np.int32)
        self.L.orc_permute(_np_ptr(np.ascontiguousarray(idx, np.int32)), T, E, k, _np_ptr(counts), _np_ptr(offsets),
                           _np_ptr(perm), _np_ptr(inv))
        return counts, offsets, perm, inv

    def ffn_bf16(self, x, M, wgu, wd, d, f):
        y = np.empty(M * d, np.float32)
        self.L.orc_ffn_bf16(_np_ptr(np.ascontiguousarray(x)), M, _np_ptr(wgu), _np_ptr(wd), d, f, _np_ptr(y))
        return y.reshape(M, d)

    def ffn_int4(self, x, M, qgu, sgu, qd, sd, d, f):
        y = np.empty(M * d, np.float32)
        self.L.orc_ffn_int4(_np_ptr(np.ascontiguousarray(x)), M, _np_ptr(qgu), _np_ptr(sgu), _np_ptr(qd),
                            _np_ptr(sd), d, f, _np_ptr(y))
        return y.reshape(M, d)

    def combine(self, y_perm, inv, w, residual, T, d, k):
        out = np.empty(T * d, np.uint16)
        self.L.orc_combine(_np_ptr(y_perm), _np_ptr(inv), _np_ptr(w), _np_ptr(residual), T, d, k, _np_ptr(out))
        return out.reshape(T, d)

    def moe_layer(self, m, layer, precision, x, T):
        out = np.empty(T * m.d_model, np.uint16)
        idx = np.empty(T * m.top_k, np.int32)
        w = np.empty(T * m.top_k, np.float32)
        lg = np.empty(T * m.num_experts, np.float32)
        prec = np.ascontiguousarray(precision, np.int32)
        self.L.orc_moe_layer(C.byref(m), layer, _np_ptr(prec), _np_ptr(np.ascontiguousarray(x)), T, _np_ptr(out),
                             _np_ptr(idx), _np_ptr(w), _np_ptr(lg))
        return out.reshape(T, m.d_model), idx.reshape(T, m.top_k), w.reshape(T, m.top_k), lg.reshape(T, m.num_experts)

    def prepare_layer(self, m, layer, precision):
        """Materialise router + the E experts of one layer (untimed setup for
        the CPU baseline).  Returns an opaque tuple for moe_layer_w."""
        keep = []
        arr = (OrcExpert * m.num_experts)()
        for s in range(m.num_experts):
            e = layer * m.num_experts + s
            if precision[s] == 1:
                gu, dn = self.expert_bf16(m, e)
                keep += [gu, dn]
                arr[s] = OrcExpert(1, _np_ptr(gu), None, _np_ptr(dn), None)
            else:
                qgu, sgu, qd, sd = self.expert_int4(m, e)
                keep += [qgu, sgu, qd, sd]
                arr[s] = OrcExpert(0, _np_ptr(qgu), _np_ptr(sgu), _np_ptr(qd), _np_ptr(sd))
        wg = self.router_weights(m, layer)
        keep.append(wg)
        return (wg, arr, keep)

    def moe_layer_w(self, m, prepared, x, T):
        wg, arr, _ = prepared
        out = np.empty(T * m.d_model, np.uint16)
        idx = np.empty(T * m.top_k, np.int32)
        self.L.orc_moe_layer_w(C.byref(m), _np_ptr(wg), arr, _np_ptr(np.ascontiguousarray(x)), T, _np_ptr(out),
                               _np_ptr(idx), None, None)
        return out.reshape(T, m.d_model), idx.reshape(T, m.top_k)

    def num_threads(self):
        return self.L.orc_num_threads()


class RefProfile(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("pad_", C.c_int32), ("size_nonexpert_bytes", C.c_int64), ("size_expert16_bytes", C.c_int64),
                ("quant_ratio", C.c_double), ("compute_latency16_s", C.c_double), ("compute_penalty4", C.c_double),
                ("nonexpert_latency_s", C.c_double)]


class RefLib:
    """The reference library itself (oracle/_ref), through ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref, needs /root/reference)")
        L = C.CDLL(path)
        I, I64, U64, D = C.c_int, C.c_int64, C.c_uint64, C.c_double
        PR = P(RefProfile)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_default_profile": (None, [I, PR]),
            "ref_load_profiles": (I, [C.c_char_p, PR, P(I64), P(D)]),
            "ref_expert_size": (I64, [PR, I]),
            "ref_model_size": (I, [PR, I, I, P(I64)]),
            "ref_profile_fingerprint": (U64, [PR]),
            "ref_num_experts_16": (I, [PR, I64]),
            "ref_make_plan": (I, [PR, I64, D, I, I, U64, VP, VP, P(I64)]),
            "ref_assign_locations": (I, [PR, I64, D, VP, U64, VP, P(I64)]),
            "ref_generate_trace": (I, [PR, I, U64, VP, P(U64)]),
            "ref_write_trace": (I64, [PR, I, VP, C.c_char_p, I64]),
            "ref_read_trace": (I, [C.c_char_p, VP, P(U64), VP, I64]),
            "ref_simulate": (I, [PR, D, VP, VP, I64, U64, I, VP, I, VP]),
            "ref_expected_throughput": (D, [PR, D, VP, VP, I64]),
            "ref_diff_plans": (I, [PR, D, VP, VP, VP, VP, VP, VP, I, P(I64), P(D)]),
            "ref_have_serialize": (I, []),
            "ref_reconfig_diff": (I, [PR, D, VP, VP, VP, VP, U64, VP, I, P(I64), P(D)]),
            "ref_reconfig_apply": (I, [PR, VP, VP, U64, VP, I, U64, I64, VP, VP, P(I64), P(U64)]),
            "ref_builtin_anchors": (I, [C.c_char_p, P(D), P(D)]),
            "ref_load_anchors": (I, [C.c_char_p, P(D), P(D)]),
            "ref_ppl_estimate": (I, [I, D, D, I, P(D)]),
            "ref_n4_for_budget": (I, [D, D, D, I, P(C.c_int32)]),
            "ref_frontier_mask": (I, [I, VP, VP, VP, VP]),
            "ref_pareto_sweep": (I, [PR, D, VP, I, VP, I, I, U64, D, D, VP]),
        }
        if L.ref_have_serialize():
            sig["ref_write_plan"] = (I64, [PR, VP, VP, U64, I64, C.c_char_p, I64])
            sig["ref_read_plan"] = (I, [C.c_char_p, PR, VP, VP, P(U64), P(I64)])
            sig["ref_write_reconfig"] = (I64, [PR, D, VP, VP, VP, VP, U64, C.c_char_p, I64])
            sig["ref_read_reconfig"] = (I, [C.c_char_p, PR, D, VP, I, P(I), P(U64), P(I64), P(D)])
            sig["ref_report_text"] = (I64, [VP, I, C.c_char_p, I64])
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        self.L = L

    def err(self):
        return self.L.ref_last_error().decode()

    @staticmethod
    def profile(p) -> RefProfile:
        return RefProfile(p.num_layers, p.experts_per_layer, p.top_k, 0, p.size_nonexpert_bytes,
                          p.size_expert16_bytes, p.quant_ratio, p.compute_latency16_s, p.compute_penalty4,
                          p.nonexpert_latency_s)

    def default_profile(self, which=0) -> RefProfile:
        r = RefProfile()
        self.L.ref_default_profile(which, C.byref(r))
        return r

    def make_plan(self, p, gpu_mem, bw, preference, n4_target, seed):
        n = p.num_layers * p.experts_per_layer
        prec = np.empty(n, np.int32)
        loc = np.empty(n, np.int32)
        swap = C.c_int64()
        st = self.L.ref_make_plan(C.byref(self.profile(p)), gpu_mem, bw, preference,
                                  -1 if n4_target is None else n4_target, seed, _np_ptr(prec), _np_ptr(loc),
                                  C.byref(swap))
        return st, prec, loc, swap.value

    def generate_trace(self, p, tokens, seed):
        n = tokens * p.num_layers * p.top_k
        slots = np.empty(n, np.int32)
        fp = C.c_uint64()
        st = self.L.ref_generate_trace(C.byref(self.profile(p)), tokens, seed, _np_ptr(slots), C.byref(fp))
        return st, slots, fp.value

    def write_trace(self, p, tokens, slots):
        arr = np.ascontiguousarray(slots, np.int32)
        n = self.L.ref_write_trace(C.byref(self.profile(p)), tokens, _np_ptr(arr), None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.L.ref_write_trace(C.byref(self.profile(p)), tokens, _np_ptr(arr), buf, n + 1)
        return buf.value.decode()

    # rows as (budget, n4, feasible, on_frontier, n_gpu, gpu_bytes, ppl,
    # tokens, activations, hits, bytes_transferred, transfer_ns, compute_ns, nonexpert_ns)
    PARETO_ROW = np.dtype([("budget", "<i8"), ("n4", "<i4"), ("feasible", "<i4"), ("on_frontier", "<i4"),
                           ("n_gpu", "<i4"), ("gpu_bytes", "<i8"), ("ppl", "<f8"), ("tokens", "<i8"),
                           ("activations", "<i8"), ("hits", "<i8"), ("bytes_transferred", "<i8"),
                           ("transfer_ns", "<i8"), ("compute_ns", "<i8"), ("nonexpert_ns", "<i8")])

    def pareto_sweep(self, p, bw, budgets, grid, tokens, seed, p16, p4):
        """sweep_memory + ppl_estimate + frontier_mask (cli.cpp:308-342)."""
        b = np.ascontiguousarray(budgets, np.int64)
        g = np.ascontiguousarray(grid, np.int32)
        rows = np.zeros(max(len(b) * len(g), 1), self.PARETO_ROW)
        st = self.L.ref_pareto_sweep(C.byref(self.profile(p)), bw, _np_ptr(b), len(b), _np_ptr(g), len(g), tokens,
                                     seed, p16, p4, rows.ctypes.data)
        return st, rows[:len(b) * len(g)]

    def ppl_estimate(self, n4, p16, p4, num_e):
        out = C.c_double()
        return self.L.ref_ppl_estimate(n4, p16, p4, num_e, C.byref(out)), out.value

    def n4_for_budget(self, budget, p16, p4, num_e):
        out = C.c_int32()
        return self.L.ref_n4_for_budget(budget, p16, p4, num_e, C.byref(out)), out.value

    def builtin_anchors(self, name):
        a, b = C.c_double(), C.c_double()
        return self.L.ref_builtin_anchors(name.encode(), C.byref(a), C.byref(b)), a.value, b.value

    def load_anchors(self, doc, p16, p4):
        a, b = C.c_double(p16), C.c_double(p4)
        return self.L.ref_load_anchors(doc.encode(), C.byref(a), C.byref(b)), a.value, b.value

    def frontier_mask(self, tps, ppl, gpu_bytes):
        t = np.ascontiguousarray(tps, np.float64)
        q = np.ascontiguousarray(ppl, np.float64)
        g = np.ascontiguousarray(gpu_bytes, np.int64)
        out = np.zeros(max(len(t), 1), np.int32)
        st = self.L.ref_frontier_mask(len(t), t.ctypes.data, q.ctypes.data, g.ctypes.data, out.ctypes.data)
        return st, out[:len(t)].astype(bool)

    def reconfig_diff(self, p, bw, prec_a, loc_a, prec_b, loc_b, seed_b=0):
        """diff_plans (reconfig.cpp:19-55): (status, [(kind, layer, slot, tprec, tloc)], bytes, downtime)."""
        arrs = [np.ascontiguousarray(v, np.int32) for v in (prec_a, loc_a, prec_b, loc_b)]
        cap = 4 * len(arrs[0]) + 4
        acts = np.zeros(5 * cap, np.int32)
        b, t = C.c_int64(), C.c_double()
        n = self.L.ref_reconfig_diff(C.byref(self.profile(p)), bw, *[_np_ptr(a) for a in arrs], seed_b, _np_ptr(acts),
                                     cap, C.byref(b), C.byref(t))
        if n < 0:
            return -n, None, None, None
        return 0, [tuple(int(v) for v in acts[5 * i:5 * i + 5]) for i in range(n)], b.value, t.value

    def reconfig_apply(self, p, prec, loc, seed, actions, target_seed, budget=0):
        """apply (reconfig.cpp:84-168): (status, prec, loc, swap, seed)."""
        n = p.num_layers * p.experts_per_layer
        a = np.ascontiguousarray(np.array(actions, np.int32).reshape(-1), np.int32) if actions else np.zeros(5, np.int32)
        op, ol = np.zeros(n, np.int32), np.zeros(n, np.int32)
        sw, sd = C.c_int64(), C.c_uint64()
        st = self.L.ref_reconfig_apply(C.byref(self.profile(p)), _np_ptr(np.ascontiguousarray(prec, np.int32)),
                                       _np_ptr(np.ascontiguousarray(loc, np.int32)), seed, _np_ptr(a), len(actions),
                                       target_seed, budget, _np_ptr(op), _np_ptr(ol), C.byref(sw), C.byref(sd))
        return st, op, ol, sw.value, sd.value

    @property
    def has_serialize(self) -> bool:
        return bool(self.L.ref_have_serialize())

    def write_plan(self, p, prec, loc, seed, swap):
        """serialize.cpp:99-117 (status, document)."""
        pr, lo = np.ascontiguousarray(prec, np.int32), np.ascontiguousarray(loc, np.int32)
        n = self.L.ref_write_plan(C.byref(self.profile(p)), _np_ptr(pr), _np_ptr(lo), seed, swap, None, 0)
        if n < 0:
            return int(-n), None
        buf = C.create_string_buffer(int(n) + 1)
        self.L.ref_write_plan(C.byref(self.profile(p)), _np_ptr(pr), _np_ptr(lo), seed, swap, buf, n + 1)
        return 0, buf.value.decode()

    def read_plan(self, doc, p):
        """serialize.cpp:119-149 (status, prec, loc, seed, swap)."""
        n = p.num_layers * p.experts_per_layer
        prec, loc = np.zeros(n, np.int32), np.zeros(n, np.int32)
        seed, swap = C.c_uint64(), C.c_int64()
        st = self.L.ref_read_plan(doc.encode(), C.byref(self.profile(p)), _np_ptr(prec), _np_ptr(loc),
                                  C.byref(seed), C.byref(swap))
        return st, prec, loc, seed.value, swap.value

    def write_reconfig(self, p, bw, prec_a, loc_a, prec_b, loc_b, seed_b=0):
        arrs = [np.ascontiguousarray(v, np.int32) for v in (prec_a, loc_a, prec_b, loc_b)]
        args = [C.byref(self.profile(p)), bw] + [_np_ptr(a) for a in arrs] + [seed_b]
        n = self.L.ref_write_reconfig(*args, None, 0)
        if n < 0:
            return int(-n), None
        buf = C.create_string_buffer(int(n) + 1)
        self.L.ref_write_reconfig(*args, buf, n + 1)
        return 0, buf.value.decode()

    def read_reconfig(self, doc, p, bw):
        """(status, [(kind, layer, slot, tprec, tloc)], target_seed, bytes, downtime)."""
        cap = 4 * p.num_layers * p.experts_per_layer + 8
        acts = np.zeros(5 * cap, np.int32)
        n, sd, b, t = C.c_int(), C.c_uint64(), C.c_int64(), C.c_double()
        st = self.L.ref_read_reconfig(doc.encode(), C.byref(self.profile(p)), bw, _np_ptr(acts), cap, C.byref(n),
                                      C.byref(sd), C.byref(b), C.byref(t))
        if st:
            return st, None, None, None, None
        return 0, [tuple(int(v) for v in acts[5 * i:5 * i + 5]) for i in range(n.value)], sd.value, b.value, t.value

    def report_text(self, counters, json=False):
        c = np.ascontiguousarray(counters, np.int64)
        n = self.L.ref_report_text(_np_ptr(c), 1 if json else 0, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        self.L.ref_report_text(_np_ptr(c), 1 if json else 0, buf, n + 1)
        return buf.value.decode()

    def simulate(self, p, bw, prec, loc, swap, tokens, slots, lru=0):
        out = np.zeros(6, np.int64)
        st = self.L.ref_simulate(C.byref(self.profile(p)), bw, _np_ptr(np.ascontiguousarray(prec, np.int32)),
                                 _np_ptr(np.ascontiguousarray(loc, np.int32)), swap, 0, tokens,
                                 _np_ptr(np.ascontiguousarray(slots, np.int32)), lru, _np_ptr(out))
        return st, out

    def expected_throughput(self, p, bw, prec, loc, swap):
        return self.L.ref_expected_throughput(C.byref(self.profile(p)), bw,
                                              _np_ptr(np.ascontiguousarray(prec, np.int32)),
                                              _np_ptr(np.ascontiguousarray(loc, np.int32)), swap)

    def num_experts_16(self, p, mem):
        return self.L.ref_num_experts_16(C.byref(self.profile(p)), mem)

    def expert_size(self, p, prec):
        return self.L.ref_expert_size(C.byref(self.profile(p)), prec)

    def fingerprint(self, p):
        return self.L.ref_profile_fingerprint(C.byref(self.profile(p)))

    def load_profiles(self, doc):
        r = RefProfile()
        mem = C.c_int64()
        bw = C.c_double()
        st = self.L.ref_load_profiles(doc.encode(), C.byref(r), C.byref(mem), C.byref(bw))
        return st, r, mem.value, bw.value


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)
