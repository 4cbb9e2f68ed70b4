"""paper_2407_14417_b200 -- B200-native MoE expert-layer hot path of arXiv 2407.14417.

Python view of the C ABI in include/moe_b200.h (libmoe_b200.so, built in-tree
for sm_100a).  Names follow the reference's operator API
(/root/reference/proj/include/moeserve): ModelProfile / HardwareProfile /
TaskRequest (profiles.hpp:29-59), make_plan (planner.hpp:71), generate_trace
(gating.hpp:33), simulate (simulator.hpp:58), plus the kernel entry points
and MoeEngine that replace the reference's cost-model stand-ins with real
sm_100a kernels.  There is no CPU fallback: kernel calls without a CUDA
device raise MoeError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOE_B200_LIB") or os.path.join(_HERE, "libmoe_b200.so")  # override: A/B builds

MOE_P4, MOE_P16 = 0, 1
MOE_GPU, MOE_CPU = 0, 1
THROUGHPUT, QUALITY = 0, 1
MAX_EXPERTS = 64


class MoeError(RuntimeError):
    """Raised for non-zero status; .code mirrors the reference CLI exit codes
    (cli.hpp:7-8): 1 internal, 2 usage, 3 parse/validation, 4 infeasible."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ValidationError(MoeError):
    pass


class InfeasibleError(MoeError):
    pass


class UsageError(MoeError):
    pass


class _ModelProfile(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("pad_", C.c_int32), ("size_nonexpert_bytes", C.c_int64),
                ("size_expert16_bytes", C.c_int64), ("quant_ratio", C.c_double),
                ("compute_latency16_s", C.c_double), ("compute_penalty4", C.c_double),
                ("nonexpert_latency_s", C.c_double)]


class _HardwareProfile(C.Structure):
    _fields_ = [("gpu_mem_bytes", C.c_int64), ("transfer_bw_bytes_per_s", C.c_double)]


class _TaskRequest(C.Structure):
    _fields_ = [("preference", C.c_int32), ("n4_target", C.c_int32), ("seed", C.c_uint64)]


class ExpertStateC(C.Structure):
    _fields_ = [("precision", C.c_int32), ("location", C.c_int32)]


class SimReportC(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("activations", C.c_int64), ("hits", C.c_int64),
                ("bytes_transferred", C.c_int64), ("transfer_ns", C.c_int64),
                ("compute_ns", C.c_int64), ("nonexpert_ns", C.c_int64)]


class ParetoRowC(C.Structure):
    _fields_ = [("budget", C.c_int64), ("n4", C.c_int32), ("feasible", C.c_int32), ("on_frontier", C.c_int32),
                ("n_gpu", C.c_int32), ("gpu_bytes", C.c_int64), ("ppl", C.c_double), ("report", SimReportC)]


class ReconfigActionC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("slot", C.c_int32), ("target_precision", C.c_int32),
                ("target_location", C.c_int32), ("pad_", C.c_int32)]


class ReconfigReportC(C.Structure):
    _fields_ = [("actions", C.c_int32), ("pad_", C.c_int32), ("bytes_moved", C.c_int64), ("est_downtime_s", C.c_double),
                ("bytes_h2d", C.c_int64), ("measured_s", C.c_double)]


class ExpertWeightsC(C.Structure):
    _fields_ = [("precision", C.c_int32), ("pad_", C.c_int32), ("w_gate_up", C.c_void_p),
                ("s_gate_up", C.c_void_p), ("w_down", C.c_void_p), ("s_down", C.c_void_p)]


class _EngineConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("d_model", C.c_int32), ("d_ffn", C.c_int32), ("max_tokens", C.c_int32),
                ("seed", C.c_uint64), ("device", C.c_int32), ("use_graphs", C.c_int32), ("norm_eps", C.c_float),
                ("tc_min_tokens", C.c_int32), ("lru_capacity", C.c_int32), ("keep_masters", C.c_int32),
                ("per_layer_decode", C.c_int32), ("ep_rank", C.c_int32), ("ep_world", C.c_int32)]


_lib = None


def lib() -> C.CDLL:
    """Load libmoe_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C paper_2407_14417_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    P, I, I64, U64, D, VP = C.POINTER, C.c_int, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
    sig = {
        "moe_last_error": (C.c_char_p, []),
        "moe_ep_last_error": (C.c_char_p, []),
        "moe_ep_unique_id": (I, [C.c_char_p]),
        "moe_ep_comm_init": (I, [C.c_char_p, I, I, I, P(VP)]),
        "moe_ep_comm_wrap": (I, [VP, I, I, P(VP)]),
        "moe_ep_comm_destroy": (None, [VP]),
        "moe_ep_dispatch": (I, [VP, VP, I, I, VP, VP]),
        "moe_ep_combine": (I, [VP, VP, I, I, VP, VP]),
        "moe_ep_peer_bytes": (C.c_size_t, [I, I, I]),
        "moe_ep_peer_rows": (VP, [VP]),
        "moe_ep_peer_alloc": (I, [C.c_size_t, P(VP)]),
        "moe_ep_peer_free": (I, [VP]),
        "moe_ep_peer_ipc_handle": (I, [VP, C.c_char_p]),
        "moe_ep_peer_ipc_open": (I, [C.c_char_p, P(VP)]),
        "moe_ep_peer_ipc_close": (I, [VP]),
        "moe_ep_push_rows": (I, [VP, I, I, I, I, P(VP), C.c_uint32, VP]),
        "moe_ep_wait_rows": (I, [VP, I, I, I, C.c_uint32, VP]),
        "moe_ep_push_shares": (I, [VP, VP, VP, VP, U64, I, I, I, I, I, P(VP), C.c_uint32, VP]),
        "moe_ep_reduce": (I, [VP, I, I, I, I, P(VP), C.c_uint32, VP, VP]),
        "moe_version": (I, []),
        "moe_profile_builtin": (I, [I, P(_ModelProfile)]),
        "moe_profile_for_shape": (I, [I, I, I, I, I, I64, P(_ModelProfile)]),
        "moe_load_profiles": (I, [C.c_char_p, P(_ModelProfile), P(_HardwareProfile)]),
        "moe_parse_size": (I64, [C.c_char_p]),
        "moe_expert_size": (I64, [P(_ModelProfile), I]),
        "moe_model_size": (I, [P(_ModelProfile), I, I, P(I64)]),
        "moe_profile_fingerprint": (U64, [P(_ModelProfile)]),
        "moe_num_experts_16": (I, [I64, P(_ModelProfile)]),
        "moe_make_plan": (I, [P(_TaskRequest), P(_HardwareProfile), P(_ModelProfile), P(ExpertStateC), P(I64)]),
        "moe_assign_locations": (I, [P(C.c_int32), P(_HardwareProfile), P(_ModelProfile), U64, P(ExpertStateC), P(I64)]),
        "moe_gpu_footprint": (I64, [P(ExpertStateC), I64, P(_ModelProfile)]),
        "moe_validate_plan": (I, [P(ExpertStateC), I, I64, P(_HardwareProfile), P(_ModelProfile), C.c_char_p, I]),
        "moe_generate_trace": (I, [P(_ModelProfile), I, U64, P(C.c_int32), P(U64)]),
        "moe_write_plan": (I64, [P(ExpertStateC), I64, U64, P(_ModelProfile), C.c_char_p, I64]),
        "moe_read_plan": (I, [C.c_char_p, P(_ModelProfile), P(ExpertStateC), P(I64), P(U64)]),
        "moe_write_trace": (I64, [P(_ModelProfile), I, P(C.c_int32), C.c_char_p, I64]),
        "moe_read_trace": (I, [C.c_char_p, P(C.c_int32), P(U64), P(C.c_int32), I64]),
        "moe_simulate": (I, [P(ExpertStateC), I64, P(C.c_int32), I, P(_ModelProfile), P(_HardwareProfile), I, P(SimReportC)]),
        "moe_expected_throughput": (D, [P(ExpertStateC), P(_ModelProfile), P(_HardwareProfile)]),
        "moe_diff_plans": (I, [P(ExpertStateC), P(ExpertStateC), U64, P(_ModelProfile), P(_HardwareProfile),
                               P(ReconfigActionC), I, P(I), P(I64), P(D)]),
        "moe_apply_reconfig": (I, [P(ExpertStateC), U64, P(ReconfigActionC), I, U64, P(_ModelProfile),
                                   P(_HardwareProfile), P(ExpertStateC), P(I64), P(U64)]),
        "moe_engine_reconfigure": (I, [VP, P(ExpertStateC), U64, D, P(ReconfigReportC)]),
        "moe_write_reconfig": (I64, [P(ReconfigActionC), I, U64, P(_ModelProfile), P(_HardwareProfile), C.c_char_p, I64]),
        "moe_read_reconfig": (I, [C.c_char_p, P(_ModelProfile), P(_HardwareProfile), P(ReconfigActionC), I, P(I), P(U64),
                                  P(I64), P(D)]),
        "moe_report_text": (I64, [P(SimReportC), I, C.c_char_p, I64]),
        "moe_builtin_anchors": (I, [C.c_char_p, P(D), P(D)]),
        "moe_load_anchors": (I, [C.c_char_p, P(D), P(D)]),
        "moe_ppl_estimate": (I, [I, D, D, I, P(D)]),
        "moe_n4_for_budget": (I, [D, D, D, I, P(C.c_int32)]),
        "moe_pareto_sweep": (I, [P(I64), I, P(C.c_int32), I, P(_ModelProfile), P(_HardwareProfile), I, U64, D, D,
                                 P(ParetoRowC)]),
        "moe_frontier_mask": (I, [I, P(D), P(D), P(I64), P(C.c_int32)]),
        "moe_pareto_csv": (I64, [P(ParetoRowC), I, P(D), C.c_char_p, I64]),
        "moe_gate_topk": (I, [VP, VP, I, I, I, I, VP, VP, VP, VP]),
        "moe_permute": (I, [VP, I, I, I, VP, VP, VP, VP, VP]),
        "moe_ffn_workspace_bytes": (C.c_size_t, [I, I, I, I, I]),
        "moe_ffn": (I, [VP, VP, VP, I, I, P(ExpertWeightsC), I, I, I, VP, C.c_size_t, VP, VP]),
        "moe_ffn_int4": (I, [VP, VP, VP, I, I, P(VP), P(VP), P(VP), P(VP), I, I, I, VP, C.c_size_t, VP, VP]),
        "moe_ffn_tc_workspace_bytes": (C.c_size_t, [I, I, I, I]),
        "moe_route": (I, [VP, VP, I, I, I, I, C.c_float, VP, VP, VP, VP, VP, VP, VP, VP, VP, VP]),
        "moe_combine_partial": (I, [VP, VP, VP, VP, C.c_uint64, I, I, I, VP, VP]),
        "moe_residual_add": (I, [VP, VP, C.c_int64, VP, VP]),
        "moe_ffn_tc": (I, [VP, VP, VP, I, I, P(ExpertWeightsC), I, I, I, VP, C.c_size_t, VP, VP]),
        "moe_ffn_bf16": (I, [VP, VP, VP, I, I, P(VP), P(VP), I, I, I, VP, C.c_size_t, VP, VP]),
        "moe_pack_bf16_blocks": (I, [VP, I, I, VP, VP]),
        "moe_gemv_max_tokens": (I, [I, I]),
        "moe_numerics_status": (I, [I, C.POINTER(C.c_uint32)]),
        "moe_combine": (I, [VP, VP, VP, VP, I, I, I, VP, VP]),
        "moe_quantize_g128": (I, [VP, I, I, VP, VP, VP]),
        "moe_synth_weight_bf16": (I, [U64, U64, I64, I, VP, VP]),
        "moe_synth_input_bf16": (I, [U64, U64, I64, VP, VP]),
        "moe_weight_shift": (I, [I]),
        "moe_stream_expert": (I, [VP, VP, C.c_size_t, VP, VP]),
        "moe_engine_create": (I, [P(_EngineConfig), P(ExpertStateC), P(VP)]),
        "moe_engine_destroy": (None, [VP]),
        "moe_engine_memory": (I, [VP, P(I64), P(I64), P(I64), P(I64)]),
        "moe_engine_input": (VP, [VP]),
        "moe_engine_output": (VP, [VP]),
        "moe_engine_stream": (VP, [VP]),
        "moe_engine_synth_input": (I, [VP, I, I]),
        "moe_engine_decode": (I, [VP, I]),
        "moe_engine_decode_host": (I, [VP, VP, I, VP]),
        "moe_engine_forward_layer": (I, [VP, I, VP, I, VP, VP, VP, VP]),
        "moe_engine_sync": (I, [VP]),
        "moe_engine_profile_step": (I, [VP, I, P(C.c_float), P(I64), P(C.c_int32)]),
        "moe_engine_profile_fused": (I, [VP, P(C.c_float), P(I64)]),
        "moe_debug_fused_trace": (I, [VP]),
        "moe_debug_engine_buffer": (I, [VP, I, P(VP), P(C.c_size_t)]),
        "moe_engine_last_routing": (I, [VP, I, P(C.c_int32)]),
        "moe_engine_counters": (I, [VP, P(SimReportC)]),
        "moe_engine_reset_counters": (I, [VP]),
        "moe_engine_expert": (I, [VP, I, I, P(ExpertWeightsC), P(C.c_int32)]),
        "moe_engine_router": (I, [VP, I, P(VP)]),
        "moe_engine_ep_buffer": (I, [VP, P(VP), P(I64)]),
        "moe_engine_ep_set_peers": (I, [VP, P(VP), I]),
        "moe_debug_gemv_trace": (I, [VP]),
        "moe_debug_layer_trace": (I, [VP, VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> List[str]:
    """Every extern "C" function declared in include/moe_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "moe_b200.h")
    text = open(hdr).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(moe_[a-z0-9_]+)\s*\(", text)))


def _check(status: int):
    if status != 0:
        msg = lib().moe_last_error().decode(errors="replace")
        cls = {2: UsageError, 3: ValidationError, 4: InfeasibleError}.get(status, MoeError)
        raise cls(status, msg)


# ----------------------------------------------------------------- profiles
@dataclass
class ModelProfile:
    """profiles.hpp:29-43 (defaults = mixtral-sec41)."""
    num_layers: int = 32
    experts_per_layer: int = 8
    top_k: int = 2
    size_nonexpert_bytes: int = 3_160_000_000
    size_expert16_bytes: int = 336_000_000
    quant_ratio: float = 4.0
    compute_latency16_s: float = 0.9 / (13.0 * 32.0 * 2.0)
    compute_penalty4: float = 1.15
    nonexpert_latency_s: float = 0.1 / 13.0

    @property
    def num_experts(self) -> int:
        return self.num_layers * self.experts_per_layer

    def _c(self) -> _ModelProfile:
        return _ModelProfile(self.num_layers, self.experts_per_layer, self.top_k, 0,
                             self.size_nonexpert_bytes, self.size_expert16_bytes, self.quant_ratio,
                             self.compute_latency16_s, self.compute_penalty4, self.nonexpert_latency_s)

    @staticmethod
    def _from_c(c: _ModelProfile) -> "ModelProfile":
        return ModelProfile(c.num_layers, c.experts_per_layer, c.top_k, c.size_nonexpert_bytes,
                            c.size_expert16_bytes, c.quant_ratio, c.compute_latency16_s,
                            c.compute_penalty4, c.nonexpert_latency_s)


@dataclass
class HardwareProfile:
    """profiles.hpp:45-52."""
    gpu_mem_bytes: int = 80_000_000_000
    transfer_bw_bytes_per_s: float = 336_000_000.0 / 0.02735

    def _c(self) -> _HardwareProfile:
        return _HardwareProfile(self.gpu_mem_bytes, self.transfer_bw_bytes_per_s)


@dataclass
class TaskRequest:
    """profiles.hpp:55-59."""
    preference: int = THROUGHPUT
    n4_target: Optional[int] = None
    seed: int = 0


def mixtral_sec41() -> ModelProfile:
    c = _ModelProfile()
    _check(lib().moe_profile_builtin(0, C.byref(c)))
    return ModelProfile._from_c(c)


def mixtral_table1() -> ModelProfile:
    c = _ModelProfile()
    _check(lib().moe_profile_builtin(1, C.byref(c)))
    return ModelProfile._from_c(c)


def profile_for_shape(d_model: int, d_ffn: int, num_layers: int, experts_per_layer: int = 8,
                      top_k: int = 2, size_nonexpert_bytes: int = 1) -> ModelProfile:
    c = _ModelProfile()
    _check(lib().moe_profile_for_shape(d_model, d_ffn, num_layers, experts_per_layer, top_k,
                                       size_nonexpert_bytes, C.byref(c)))
    return ModelProfile._from_c(c)


def load_profiles(document: str):
    m, h = _ModelProfile(), _HardwareProfile()
    _check(lib().moe_load_profiles(document.encode(), C.byref(m), C.byref(h)))
    return ModelProfile._from_c(m), HardwareProfile(h.gpu_mem_bytes, h.transfer_bw_bytes_per_s)


def parse_size(text: str) -> int:
    v = lib().moe_parse_size(text.encode())
    if v < 0:
        _check(3)
    return v


def expert_size(profile: ModelProfile, precision: int) -> int:
    return lib().moe_expert_size(C.byref(profile._c()), precision)


def model_size(profile: ModelProfile, n4: int, nonexpert_precision: int) -> int:
    out = C.c_int64()
    _check(lib().moe_model_size(C.byref(profile._c()), n4, nonexpert_precision, C.byref(out)))
    return out.value


def profile_fingerprint(profile: ModelProfile) -> int:
    return lib().moe_profile_fingerprint(C.byref(profile._c()))


def num_experts_16(mem_gpu: int, profile: ModelProfile) -> int:
    return lib().moe_num_experts_16(mem_gpu, C.byref(profile._c()))


# ----------------------------------------------------------------- planner
@dataclass
class PlacementPlan:
    """planner.hpp:31-36: entries[layer*E + slot] = (precision, location)."""
    precision: List[int]
    location: List[int]
    swap_slot_bytes: int
    seed: int = 0

    def _entries(self):
        arr = (ExpertStateC * len(self.precision))()
        for i, (p, l) in enumerate(zip(self.precision, self.location)):
            arr[i].precision, arr[i].location = p, l
        return arr

    @property
    def n4(self) -> int:
        return sum(1 for p in self.precision if p == MOE_P4)

    @property
    def n_gpu(self) -> int:
        return sum(1 for l in self.location if l == MOE_GPU)


def make_plan(task: TaskRequest, hw: HardwareProfile, profile: ModelProfile) -> PlacementPlan:
    n = profile.num_experts
    arr = (ExpertStateC * n)()
    swap = C.c_int64()
    t = _TaskRequest(task.preference, -1 if task.n4_target is None else task.n4_target, task.seed)
    _check(lib().moe_make_plan(C.byref(t), C.byref(hw._c()), C.byref(profile._c()), arr, C.byref(swap)))
    return PlacementPlan([a.precision for a in arr], [a.location for a in arr], swap.value, task.seed)


def assign_locations(precisions: Sequence[int], hw: HardwareProfile, profile: ModelProfile,
                     seed: int = 0) -> PlacementPlan:
    n = profile.num_experts
    prec = (C.c_int32 * n)(*precisions)
    arr = (ExpertStateC * n)()
    swap = C.c_int64()
    _check(lib().moe_assign_locations(prec, C.byref(hw._c()), C.byref(profile._c()), seed, arr, C.byref(swap)))
    return PlacementPlan([a.precision for a in arr], [a.location for a in arr], swap.value, seed)


def gpu_footprint(plan: PlacementPlan, profile: ModelProfile) -> int:
    return lib().moe_gpu_footprint(plan._entries(), plan.swap_slot_bytes, C.byref(profile._c()))


def validate_plan(plan: PlacementPlan, hw: HardwareProfile, profile: ModelProfile) -> List[str]:
    buf = C.create_string_buffer(4096)
    n = lib().moe_validate_plan(plan._entries(), len(plan.precision), plan.swap_slot_bytes,
                                C.byref(hw._c()), C.byref(profile._c()), buf, 4096)
    if n < 0:
        _check(1)
    return [s for s in buf.value.decode().split("\n") if s][:n]


def write_plan(plan: PlacementPlan, profile: ModelProfile) -> str:
    """`moeserve.plan.v1` JSON, byte-identical to serialize.cpp:99-117."""
    ent = plan._entries()
    n = lib().moe_write_plan(ent, plan.swap_slot_bytes, plan.seed, C.byref(profile._c()), None, 0)
    if n < 0:
        _check(1)
    buf = C.create_string_buffer(n + 1)
    lib().moe_write_plan(ent, plan.swap_slot_bytes, plan.seed, C.byref(profile._c()), buf, n + 1)
    return buf.value.decode()


def read_plan(document: str, profile: ModelProfile) -> PlacementPlan:
    """Parse and check a plan document against `profile` (serialize.cpp:119-149)."""
    arr = (ExpertStateC * profile.num_experts)()
    swap, seed = C.c_int64(), C.c_uint64()
    _check(lib().moe_read_plan(document.encode(), C.byref(profile._c()), arr, C.byref(swap), C.byref(seed)))
    return PlacementPlan([a.precision for a in arr], [a.location for a in arr], swap.value, seed.value)


# ----------------------------------------------------------------- traces / simulate
def generate_trace(profile: ModelProfile, tokens: int, seed: int):
    n = tokens * profile.num_layers * profile.top_k
    slots = (C.c_int32 * max(n, 1))()
    fp = C.c_uint64()
    _check(lib().moe_generate_trace(C.byref(profile._c()), tokens, seed, slots, C.byref(fp)))
    return list(slots[:n]), fp.value


def write_trace(profile: ModelProfile, tokens: int, slots: Sequence[int]) -> str:
    arr = (C.c_int32 * len(slots))(*slots)
    n = lib().moe_write_trace(C.byref(profile._c()), tokens, arr, None, 0)
    if n < 0:
        _check(1)
    buf = C.create_string_buffer(n + 1)
    lib().moe_write_trace(C.byref(profile._c()), tokens, arr, buf, n + 1)
    return buf.value.decode()


def read_trace(document: str):
    dims = (C.c_int32 * 4)()
    fp = C.c_uint64()
    _check(lib().moe_read_trace(document.encode(), dims, C.byref(fp), None, 0))
    n = dims[0] * dims[1] * dims[3]
    slots = (C.c_int32 * max(n, 1))()
    _check(lib().moe_read_trace(document.encode(), dims, C.byref(fp), slots, n))
    return {"tokens": dims[0], "num_layers": dims[1], "experts_per_layer": dims[2], "top_k": dims[3],
            "fingerprint": fp.value, "slots": list(slots[:n])}


@dataclass
class SimReport:
    """simulator.hpp:33-53."""
    tokens: int = 0
    activations: int = 0
    hits: int = 0
    bytes_transferred: int = 0
    transfer_ns: int = 0
    compute_ns: int = 0
    nonexpert_ns: int = 0

    @staticmethod
    def _from_c(c: SimReportC) -> "SimReport":
        return SimReport(c.tokens, c.activations, c.hits, c.bytes_transferred, c.transfer_ns,
                         c.compute_ns, c.nonexpert_ns)

    @property
    def total_ns(self) -> int:
        return self.transfer_ns + self.compute_ns + self.nonexpert_ns

    @property
    def throughput_tps(self) -> float:
        return self.tokens / (self.total_ns / 1e9)

    @property
    def hit_rate(self) -> float:
        return 1.0 if self.activations == 0 else self.hits / self.activations


def simulate(plan: PlacementPlan, slots: Sequence[int], tokens: int, profile: ModelProfile,
             hw: HardwareProfile, lru_capacity: int = 0) -> SimReport:
    arr = (C.c_int32 * len(slots))(*slots)
    out = SimReportC()
    _check(lib().moe_simulate(plan._entries(), plan.swap_slot_bytes, arr, tokens, C.byref(profile._c()),
                              C.byref(hw._c()), lru_capacity, C.byref(out)))
    return SimReport._from_c(out)


def expected_throughput(plan: PlacementPlan, profile: ModelProfile, hw: HardwareProfile) -> float:
    return lib().moe_expected_throughput(plan._entries(), C.byref(profile._c()), C.byref(hw._c()))


# ----------------------------------------------------------------- expert-parallel exchange
def _ep_check(status: int):
    if status != 0:
        msg = lib().moe_ep_last_error().decode(errors="replace")
        raise (UsageError if status == 2 else MoeError)(status, msg)


def ep_unique_id() -> bytes:
    """ncclGetUniqueId (on one rank; broadcast it to the others)."""
    buf = C.create_string_buffer(128)
    _ep_check(lib().moe_ep_unique_id(buf))
    return buf.raw


class EpComm:
    """NCCL communicator of the C-ABI EP exchange (moe_ep_dispatch / moe_ep_combine)."""

    def __init__(self, unique_id: bytes, world: int, rank: int, device: int = 0):
        h = C.c_void_p()
        _ep_check(lib().moe_ep_comm_init(C.create_string_buffer(unique_id, 128), world, rank, device, C.byref(h)))
        self._h, self.world, self.rank = h, world, rank

    def dispatch(self, x_local, T_local: int, d: int, x_all, stream=None):
        """All-gather of bf16 token rows: x_all[world*T_local][d]."""
        _ep_check(lib().moe_ep_dispatch(self._h, _ptr(x_local), T_local, d, _ptr(x_all), stream))

    def combine(self, part, T_local: int, d: int, mine, stream=None):
        """Reduce-scatter of fp32 shares: mine[T_local][d] = sum over ranks."""
        _ep_check(lib().moe_ep_combine(self._h, _ptr(part), T_local, d, _ptr(mine), stream))

    def close(self):
        if getattr(self, "_h", None):
            lib().moe_ep_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ep_peer_bytes(G: int, T_local: int, d: int) -> int:
    return lib().moe_ep_peer_bytes(G, T_local, d)


def ep_peer_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    _check(lib().moe_ep_peer_alloc(nbytes, C.byref(p)))
    return p.value


def ep_peer_free(base_ptr: int):
    _check(lib().moe_ep_peer_free(base_ptr))


def ep_peer_ipc_handle(base_ptr: int) -> bytes:
    buf = C.create_string_buffer(64)
    _check(lib().moe_ep_peer_ipc_handle(base_ptr, buf))
    return buf.raw


def ep_peer_ipc_open(handle: bytes) -> int:
    p = C.c_void_p()
    _check(lib().moe_ep_peer_ipc_open(C.create_string_buffer(handle, 64), C.byref(p)))
    return p.value


class PeerBases:
    """The G exchange-buffer base pointers of moe_ep_push_rows & co."""

    def __init__(self, ptrs):
        self.G = len(ptrs)
        self.arr = (C.c_void_p * self.G)(*ptrs)


def ep_push_rows(x_local, T_local: int, d: int, rank: int, bases: PeerBases, epoch: int, stream=None):
    _check(lib().moe_ep_push_rows(_ptr(x_local), T_local, d, rank, bases.G, bases.arr, epoch, stream))


def ep_wait_rows(my_base: int, G: int, T_local: int, d: int, epoch: int, stream=None):
    _check(lib().moe_ep_wait_rows(my_base, G, T_local, d, epoch, stream))


def ep_push_shares(y, inv, w, idx, mask: int, T_local: int, d: int, k: int, rank: int, bases: PeerBases, epoch: int,
                   stream=None):
    _check(lib().moe_ep_push_shares(_ptr(y), _ptr(inv), _ptr(w), _ptr(idx), mask, T_local, d, k, rank, bases.G,
                                    bases.arr, epoch, stream))


def ep_reduce(x_local, T_local: int, d: int, rank: int, bases: PeerBases, epoch: int, out, stream=None):
    _check(lib().moe_ep_reduce(_ptr(x_local), T_local, d, rank, bases.G, bases.arr, epoch, _ptr(out), stream))


# ----------------------------------------------------------------- reconfiguration (f1)
OFFLOAD, FETCH, QUANTIZE, DEQUANTIZE = 0, 1, 2, 3


def diff_plans(src: PlacementPlan, dst: PlacementPlan, profile: ModelProfile, hw: HardwareProfile):
    """reconfig.cpp:19-55: ([(kind, layer, slot, target_precision, target_location)], bytes_moved, est_downtime_s)."""
    n = profile.num_experts
    cap = 2 * n
    acts = (ReconfigActionC * cap)()
    cnt, b, t = C.c_int(), C.c_int64(), C.c_double()
    _check(lib().moe_diff_plans(src._entries(), dst._entries(), dst.seed, C.byref(profile._c()), C.byref(hw._c()), acts,
                                cap, C.byref(cnt), C.byref(b), C.byref(t)))
    return ([(a.kind, a.layer, a.slot, a.target_precision, a.target_location) for a in acts[:cnt.value]], b.value,
            t.value)


def apply_reconfig(plan: PlacementPlan, actions, target_seed: int, profile: ModelProfile,
                   budget: HardwareProfile = None) -> PlacementPlan:
    """reconfig.cpp:84-168: checked replay of an action list."""
    acts = (ReconfigActionC * max(len(actions), 1))(*[ReconfigActionC(*a, 0) for a in actions])
    out = (ExpertStateC * profile.num_experts)()
    sw, sd = C.c_int64(), C.c_uint64()
    _check(lib().moe_apply_reconfig(plan._entries(), plan.seed, acts, len(actions), target_seed, C.byref(profile._c()),
                                    C.byref(budget._c()) if budget is not None else None, out, C.byref(sw),
                                    C.byref(sd)))
    return PlacementPlan([a.precision for a in out], [a.location for a in out], sw.value, sd.value)


def write_reconfig(actions, target_seed: int, profile: ModelProfile, hw: HardwareProfile) -> str:
    """moeserve.reconfig.v1 JSON, byte-identical to serialize.cpp:160-176."""
    acts = (ReconfigActionC * max(len(actions), 1))(*[ReconfigActionC(*a, 0) for a in actions])
    args = (acts, len(actions), target_seed, C.byref(profile._c()), C.byref(hw._c()))
    n = lib().moe_write_reconfig(*args, None, 0)
    if n < 0:
        _check(1)
    buf = C.create_string_buffer(n + 1)
    lib().moe_write_reconfig(*args, buf, n + 1)
    return buf.value.decode()


def read_reconfig(document: str, profile: ModelProfile, hw: HardwareProfile):
    """serialize.cpp:178-206: (actions, target_seed, bytes_moved, est_downtime_s)."""
    cap = 4 * profile.num_experts + 8
    acts = (ReconfigActionC * cap)()
    n, sd, b, t = C.c_int(), C.c_uint64(), C.c_int64(), C.c_double()
    _check(lib().moe_read_reconfig(document.encode(), C.byref(profile._c()), C.byref(hw._c()), acts, cap, C.byref(n),
                                   C.byref(sd), C.byref(b), C.byref(t)))
    return ([(a.kind, a.layer, a.slot, a.target_precision, a.target_location) for a in acts[:n.value]], sd.value,
            b.value, t.value)


def report_text(report: "SimReport", json: bool = False) -> str:
    """The reference's report_csv / report_json (serialize.cpp:218-243)."""
    r = SimReportC(report.tokens, report.activations, report.hits, report.bytes_transferred, report.transfer_ns,
                   report.compute_ns, report.nonexpert_ns)
    n = lib().moe_report_text(C.byref(r), 1 if json else 0, None, 0)
    if n < 0:
        _check(1)
    buf = C.create_string_buffer(n + 1)
    lib().moe_report_text(C.byref(r), 1 if json else 0, buf, n + 1)
    return buf.value.decode()


# ----------------------------------------------------------------- pareto (f3)
@dataclass
class QualityAnchors:
    """pareto.hpp:14-19; defaults = wikitext2 (Table 2)."""
    ppl_all16: float = 3.81
    ppl_all4: float = 4.00


def builtin_anchors(name: str) -> QualityAnchors:
    a, b = C.c_double(), C.c_double()
    _check(lib().moe_builtin_anchors(name.encode(), C.byref(a), C.byref(b)))
    return QualityAnchors(a.value, b.value)


def load_anchors(document: str, fallback: QualityAnchors = None) -> QualityAnchors:
    fallback = fallback or QualityAnchors()
    a, b = C.c_double(fallback.ppl_all16), C.c_double(fallback.ppl_all4)
    _check(lib().moe_load_anchors(document.encode(), C.byref(a), C.byref(b)))
    return QualityAnchors(a.value, b.value)


def ppl_estimate(n4: int, anchors: QualityAnchors, num_e: int) -> float:
    out = C.c_double()
    _check(lib().moe_ppl_estimate(n4, anchors.ppl_all16, anchors.ppl_all4, num_e, C.byref(out)))
    return out.value


def n4_for_budget(ppl_budget: float, anchors: QualityAnchors, num_e: int) -> int:
    out = C.c_int32()
    _check(lib().moe_n4_for_budget(ppl_budget, anchors.ppl_all16, anchors.ppl_all4, num_e, C.byref(out)))
    return out.value


def frontier_mask(throughput_tps: Sequence[float], ppl: Sequence[float], gpu_bytes: Sequence[int]) -> List[bool]:
    n = len(throughput_tps)
    out = (C.c_int32 * max(n, 1))()
    _check(lib().moe_frontier_mask(n, (C.c_double * max(n, 1))(*throughput_tps), (C.c_double * max(n, 1))(*ppl),
                                   (C.c_int64 * max(n, 1))(*gpu_bytes), out))
    return [bool(v) for v in out[:n]]


@dataclass
class ParetoRow:
    """cli.cpp:243-251: one (budget, n4) cell; `report` is the Static simulate."""
    budget: int
    n4: int
    feasible: bool
    on_frontier: bool
    n_gpu: int
    gpu_bytes: int
    ppl: float
    report: SimReport

    def _c(self) -> ParetoRowC:
        r = self.report
        return ParetoRowC(self.budget, self.n4, int(self.feasible), int(self.on_frontier), self.n_gpu,
                          self.gpu_bytes, self.ppl,
                          SimReportC(r.tokens, r.activations, r.hits, r.bytes_transferred, r.transfer_ns,
                                     r.compute_ns, r.nonexpert_ns))


def pareto_sweep(budgets: Sequence[int], n4_grid: Sequence[int], profile: ModelProfile, hw: HardwareProfile,
                 tokens: int = 2000, seed: int = 0, anchors: QualityAnchors = None) -> List[ParetoRow]:
    """Rows for n4_grid x budgets (grid-major), frontier flags set (cli.cpp:308-342)."""
    anchors = anchors or QualityAnchors()
    nb, ng = len(budgets), len(n4_grid)
    rows = (ParetoRowC * max(nb * ng, 1))()
    _check(lib().moe_pareto_sweep((C.c_int64 * max(nb, 1))(*budgets), nb, (C.c_int32 * max(ng, 1))(*n4_grid), ng,
                                  C.byref(profile._c()), C.byref(hw._c()), tokens, seed, anchors.ppl_all16,
                                  anchors.ppl_all4, rows))
    return [ParetoRow(r.budget, r.n4, bool(r.feasible), bool(r.on_frontier), r.n_gpu, r.gpu_bytes, r.ppl,
                      SimReport._from_c(r.report)) for r in rows[:nb * ng]]


def pareto_csv(rows: Sequence[ParetoRow], measured: Sequence = None) -> str:
    """The reference sweep table (cli.cpp:253-270); `measured` = per-row
    (tok/s, hit rate) or None appends measured_tps,measured_hit_rate."""
    n = len(rows)
    arr = (ParetoRowC * max(n, 1))(*[r._c() for r in rows])
    meas = None
    if measured is not None:
        flat = []
        for m in measured:
            flat.extend((float("nan"), float("nan")) if m is None else (float(m[0]), float(m[1])))
        meas = (C.c_double * max(len(flat), 1))(*flat)
    k = lib().moe_pareto_csv(arr, n, meas, None, 0)
    if k < 0:
        _check(1)
    buf = C.create_string_buffer(k + 1)
    lib().moe_pareto_csv(arr, n, meas, buf, k + 1)
    return buf.value.decode()


# ----------------------------------------------------------------- kernels
def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


def _stream(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:
            return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def gate_topk(x, wg, T, d, E, k, idx, w, logits=None, stream=None):
    _check(lib().moe_gate_topk(_ptr(x), _ptr(wg), T, d, E, k, _ptr(idx), _ptr(w), _ptr(logits), _stream(stream)))


def permute(idx, T, E, k, counts, offsets, perm, inv_perm, stream=None):
    _check(lib().moe_permute(_ptr(idx), T, E, k, _ptr(counts), _ptr(offsets), _ptr(perm), _ptr(inv_perm),
                             _stream(stream)))


def expert_weights(precision, w_gate_up, w_down, s_gate_up=None, s_down=None) -> ExpertWeightsC:
    return ExpertWeightsC(precision, 0, _ptr(w_gate_up), _ptr(s_gate_up), _ptr(w_down), _ptr(s_down))


def ffn_workspace_bytes(T, k, E, d, f) -> int:
    return lib().moe_ffn_workspace_bytes(T, k, E, d, f)


def ffn(x, perm, offsets, T, k, experts: Sequence[ExpertWeightsC], d, f, workspace, ws_bytes, y_perm,
        stream=None):
    """K3/K4 grouped SwiGLU FFN; `workspace` (ffn_workspace_bytes) zero-filled once."""
    arr = (ExpertWeightsC * len(experts))(*experts)
    _check(lib().moe_ffn(_ptr(x), _ptr(perm), _ptr(offsets), T, k, arr, len(experts), d, f, _ptr(workspace),
                         ws_bytes, _ptr(y_perm), _stream(stream)))


NUMERICS_F16_ACTIVATION = 1
NUMERICS_F16_SCALE = 2


def numerics_status(clear: bool = True) -> int:
    """fp16-operand range guard bits (moe_numerics_status); sticky until cleared."""
    v = C.c_uint32()
    _check(lib().moe_numerics_status(1 if clear else 0, C.byref(v)))
    return v.value


def route(x, wg, T, d, E, k, norm_eps, idx, w, logits=None, counts=None, offsets=None, perm=None, inv_perm=None,
          xnat=None, ticket=None, stream=None):
    """K1+K2 fused (RMSNorm -> router -> top-k -> stable permutation)."""
    _check(lib().moe_route(_ptr(x), _ptr(wg), T, d, E, k, C.c_float(norm_eps), _ptr(idx), _ptr(w), _ptr(logits),
                           _ptr(counts), _ptr(offsets), _ptr(perm), _ptr(inv_perm), _ptr(xnat), _ptr(ticket),
                           _stream(stream)))


def combine_partial(y_perm, inv_perm, w, idx, expert_mask, T, d, k, out, stream=None):
    _check(lib().moe_combine_partial(_ptr(y_perm), _ptr(inv_perm), _ptr(w), _ptr(idx), expert_mask, T, d, k,
                                     _ptr(out), _stream(stream)))


def residual_add(residual, part, n, out, stream=None):
    _check(lib().moe_residual_add(_ptr(residual), _ptr(part), n, _ptr(out), _stream(stream)))


def ffn_tc_workspace_bytes(T, k, d, f) -> int:
    return lib().moe_ffn_tc_workspace_bytes(T, k, d, f)


def ffn_tc(x, perm, offsets, T, k, experts: Sequence[ExpertWeightsC], d, f, workspace, ws_bytes, y_perm,
           stream=None):
    """K3/K4 grouped SwiGLU FFN on tcgen05 (batched decode / prefill)."""
    arr = (ExpertWeightsC * len(experts))(*experts)
    _check(lib().moe_ffn_tc(_ptr(x), _ptr(perm), _ptr(offsets), T, k, arr, len(experts), d, f, _ptr(workspace),
                            ws_bytes, _ptr(y_perm), _stream(stream)))


def pack_bf16_blocks(w, rows, cols, out, stream=None):
    _check(lib().moe_pack_bf16_blocks(_ptr(w), rows, cols, _ptr(out), _stream(stream)))


def combine(y_perm, inv_perm, w, residual, T, d, k, out, stream=None):
    _check(lib().moe_combine(_ptr(y_perm), _ptr(inv_perm), _ptr(w), _ptr(residual), T, d, k, _ptr(out),
                             _stream(stream)))


def quantize_g128(w, rows, cols, q, s, stream=None):
    _check(lib().moe_quantize_g128(_ptr(w), rows, cols, _ptr(q), _ptr(s), _stream(stream)))


def synth_weight_bf16(seed, uid, n, shift, out, stream=None):
    _check(lib().moe_synth_weight_bf16(seed, uid, n, shift, _ptr(out), _stream(stream)))


def weight_shift(K: int) -> int:
    return lib().moe_weight_shift(K)


# ----------------------------------------------------------------- engine
class MoeEngine:
    """One MoE layer stack on one device (include/moeb200/engine.hpp)."""

    def __init__(self, num_layers: int, experts_per_layer: int, top_k: int, d_model: int, d_ffn: int,
                 plan: PlacementPlan, max_tokens: int = 1, seed: int = 0, device: int = 0,
                 use_graphs: bool = True, norm_eps: float = 0.0, tc_min_tokens: int = 0, lru_capacity: int = 0,
                 keep_masters: bool = False, per_layer_decode: bool = False, ep_rank: int = 0, ep_world: int = 1):
        self.L, self.E, self.k, self.d, self.f = num_layers, experts_per_layer, top_k, d_model, d_ffn
        self.ep_rank, self.ep_world = ep_rank, ep_world
        self.max_tokens = max_tokens
        self.norm_eps = norm_eps
        cfg = _EngineConfig(num_layers, experts_per_layer, top_k, d_model, d_ffn, max_tokens, seed, device,
                            1 if use_graphs else 0, norm_eps, tc_min_tokens, lru_capacity, 1 if keep_masters else 0,
                            1 if per_layer_decode else 0, ep_rank, ep_world)
        h = C.c_void_p()
        _check(lib().moe_engine_create(C.byref(cfg), plan._entries(), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().moe_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def input_ptr(self) -> int:
        return lib().moe_engine_input(self._h)

    @property
    def output_ptr(self) -> int:
        return lib().moe_engine_output(self._h)

    @property
    def stream_ptr(self) -> int:
        return lib().moe_engine_stream(self._h)

    def memory(self):
        vals = [C.c_int64() for _ in range(4)]
        _check(lib().moe_engine_memory(self._h, *[C.byref(v) for v in vals]))
        return dict(zip(["expert_bytes", "swap_bytes", "host_pinned_bytes", "workspace_bytes"],
                        [v.value for v in vals]))

    def synth_input(self, step: int, T: int):
        _check(lib().moe_engine_synth_input(self._h, step, T))

    def decode(self, T: int):
        _check(lib().moe_engine_decode(self._h, T))

    def decode_host(self, x_host_ptr: int, T: int, out_host_ptr: int):
        _check(lib().moe_engine_decode_host(self._h, x_host_ptr, T, out_host_ptr))

    def forward_layer(self, layer, x, T, out, idx=None, w=None, logits=None):
        _check(lib().moe_engine_forward_layer(self._h, layer, _ptr(x), T, _ptr(out), _ptr(idx), _ptr(w),
                                              _ptr(logits)))

    def sync(self):
        _check(lib().moe_engine_sync(self._h))

    def ep_buffer(self):
        """(device pointer, bytes) of this rank's expert-parallel exchange buffer."""
        p, n = C.c_void_p(), C.c_int64()
        _check(lib().moe_engine_ep_buffer(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def ep_set_peers(self, bases):
        """Exchange-buffer bases of all ranks in rank order (this one's included)."""
        arr = (C.c_void_p * len(bases))(*bases)
        _check(lib().moe_engine_ep_set_peers(self._h, arr, len(bases)))

    def profile_step(self, T: int):
        """Per-layer expert-FFN milliseconds (CUDA events on the launch stream),
        per-layer algorithmic bytes, kernels per decode step."""
        ms = (C.c_float * self.L)()
        by = (C.c_int64 * self.L)()
        kps = C.c_int32()
        _check(lib().moe_engine_profile_step(self._h, T, ms, by, C.byref(kps)))
        return list(ms), list(by), kps.value

    def profile_fused(self):
        """The fused batch-1 step timed alone: (ms, algorithmic bytes) or None
        when this engine decodes batch 1 layer by layer."""
        ms, by = C.c_float(), C.c_int64()
        st = lib().moe_engine_profile_fused(self._h, C.byref(ms), C.byref(by))
        if st == 2:
            return None
        _check(st)
        return ms.value, by.value

    def reconfigure(self, target: PlacementPlan, transfer_bw_bytes_per_s: float) -> dict:
        """Execute diff_plans(current, target) on the device (needs keep_masters)."""
        r = ReconfigReportC()
        _check(lib().moe_engine_reconfigure(self._h, target._entries(), target.seed, transfer_bw_bytes_per_s,
                                            C.byref(r)))
        return {"actions": r.actions, "bytes_moved": r.bytes_moved, "est_downtime_s": r.est_downtime_s,
                "bytes_h2d": r.bytes_h2d, "measured_s": r.measured_s}

    def last_routing(self, T: int) -> List[int]:
        n = T * self.L * self.k
        arr = (C.c_int32 * n)()
        _check(lib().moe_engine_last_routing(self._h, T, arr))
        return list(arr)

    def counters(self) -> SimReport:
        out = SimReportC()
        _check(lib().moe_engine_counters(self._h, C.byref(out)))
        return SimReport._from_c(out)

    def reset_counters(self):
        _check(lib().moe_engine_reset_counters(self._h))

    def expert(self, layer: int, slot: int):
        out = ExpertWeightsC()
        loc = C.c_int32()
        _check(lib().moe_engine_expert(self._h, layer, slot, C.byref(out), C.byref(loc)))
        return out, loc.value

    def router(self, layer: int) -> int:
        p = C.c_void_p()
        _check(lib().moe_engine_router(self._h, layer, C.byref(p)))
        return p.value
