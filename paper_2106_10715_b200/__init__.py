"""paper_2106_10715_b200 — B200-native InfMoE MoE-layer hot path.

Thin ctypes binding over the C-ABI library ``_lib/libinfmoe.so`` (declared in
``include/infmoe.h``).  It mirrors the reference ``moesim`` API for the
planning layer (same names, argument meaning and error behaviour:
ConfigError / CapacityError / InvariantError, std::invalid_argument ->
ValueError) and exposes the device path (gate, dispatch, expert FFN, combine,
offloaded layer handle) over raw device pointers.

There is no CPU fallback: importing raises if the CUDA library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libinfmoe.so"

if not _LIB_PATH.exists():
    raise ImportError(
        f"libinfmoe.so not built at {_LIB_PATH}; run `python -m paper_2106_10715_b200.build` "
        "(this package has no CPU fallback)")
_lib = C.CDLL(str(_LIB_PATH))

# ----------------------------------------------------------------- errors --


class ConfigError(RuntimeError):
    """moesim::ConfigError (errors.hpp:9-11), status 2."""


class CapacityError(RuntimeError):
    """moesim::CapacityError (errors.hpp:14-16), status 3."""


class InvariantError(RuntimeError):
    """moesim::InvariantError (errors.hpp:19-21), status 4."""


class CudaError(RuntimeError):
    """CUDA / NCCL runtime failure, status 5."""


class InvalidArgument(ValueError):
    """std::invalid_argument (e.g. scheduler.hpp:49-62, :74), status 6."""


_lib.infmoe_last_error.restype = C.c_char_p
_lib.infmoe_version.restype = C.c_char_p


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.infmoe_last_error() or b"").decode()
    raise {2: ConfigError, 3: CapacityError, 4: InvariantError, 5: CudaError,
                6: InvalidArgument}.get(
        rc, RuntimeError)(msg)


def version() -> str:
    return _lib.infmoe_version().decode()


def library_path() -> str:
    return str(_LIB_PATH)


# ------------------------------------------------------------------ PODs --


class Geometry(C.Structure):
    """moesim::ModelGeometry (model_config.hpp:14-22)."""
    _fields_ = [(n, C.c_int32) for n in ("n_layers", "n_heads", "d_head", "d_model", "d_ff",
                                         "n_experts_per_layer", "bytes_per_param")]


class Hardware(C.Structure):
    """moesim::HardwareProfile (model_config.hpp:27-32)."""
    _fields_ = [("peak_flops", C.c_double), ("h2d_bandwidth", C.c_double),
                ("device_memory", C.c_uint64), ("reserved_memory", C.c_uint64)]


class _ConstraintReport(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("position", C.c_int32), ("bound", C.c_int32),
                ("prefix_sum", C.c_double), ("limit", C.c_double)]


class _ScheduleInfo(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("diagnosis", C.c_int32), ("method", C.c_int32)]


class Event(C.Structure):
    """moesim::TimelineEvent (simulator.hpp:19-25); stream 0 load, 1 compute."""
    _fields_ = [("stream", C.c_int32), ("layer_id", C.c_int32), ("expert_id", C.c_int32),
                ("start", C.c_double), ("end", C.c_double)]


class _SimReport(C.Structure):
    _fields_ = [("makespan", C.c_double), ("compute_busy", C.c_double),
                ("load_busy", C.c_double), ("compute_stall", C.c_double),
                ("peak_resident_experts", C.c_int32), ("overlap_efficiency", C.c_double)]


class _LayerReport(C.Structure):
    _fields_ = [("layer_id", C.c_int32), ("n_experts", C.c_int32), ("start", C.c_double),
                ("end", C.c_double), ("compute_busy", C.c_double), ("load_busy", C.c_double),
                ("compute_stall", C.c_double), ("peak_resident", C.c_int32),
                ("lower_bound", C.c_double)]


class LayerDesc(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("d_ff", C.c_int32), ("n_experts", C.c_int32),
                ("top_k", C.c_int32), ("dtype", C.c_int32), ("gate_kind", C.c_int32),
                ("residency", C.c_int32), ("K", C.c_int32), ("policy", C.c_int32),
                ("max_tokens", C.c_int32), ("device", C.c_int32),
                ("gate_weight", C.c_void_p), ("gate_bias", C.c_void_p),
                ("lsh_seed", C.c_uint64), ("lsh_bits", C.c_int32),
                ("w_in", C.c_void_p), ("w_out", C.c_void_p), ("hw", Hardware),
                ("ep_size", C.c_int32), ("ep_rank", C.c_int32), ("ep_comm", C.c_void_p),
                ("skip_empty_experts", C.c_int32), ("slot_pool", C.c_void_p),
                ("ep_transport", C.c_int32), ("h2d_codec", C.c_int32),
                ("continuous_load_stream", C.c_int32), ("prefetch_depth", C.c_int32)]


class ForwardOut(C.Structure):
    _fields_ = [("counts", C.c_void_p), ("order", C.c_void_p), ("feasible", C.c_void_p),
                ("events", C.c_void_p), ("exposed_copy_s", C.c_void_p),
                ("local_rows", C.c_void_p), ("topk_idx", C.c_void_p), ("topk_w", C.c_void_p),
                ("perm", C.c_void_p), ("offsets", C.c_void_p), ("time_origin", C.c_void_p),
                ("prefetched", C.c_void_p)]


DTYPE_BF16, DTYPE_F32 = 0, 1
GATE_SOFTMAX, GATE_LSH = 0, 1
RESIDENT, OFFLOADED = 0, 1
POLICY_AUTO, POLICY_GREEDY, POLICY_EXACT, POLICY_NAIVE = 0, 1, 2, 3
EP_NCCL, EP_PEER = 0, 1
DIAG = {-1: None, 0: "feasible", 1: "too_little_compute", 2: "imbalanced"}
METHOD = {0: "greedy", 1: "exact_fallback", 2: "naive"}

_u64, _i32, _f64 = C.c_uint64, C.c_int32, C.c_double
_vp = C.c_void_p
_P = C.POINTER

_lib.infmoe_expert_param_bytes.restype = _u64
_lib.infmoe_expert_flops.restype = _u64
_lib.infmoe_splitmix64.restype = _u64
_lib.infmoe_splitmix64.argtypes = [_u64]
_lib.infmoe_derive_seed.restype = _u64
_lib.infmoe_derive_seed.argtypes = [_u64, _u64]
_lib.infmoe_expert_flops.argtypes = [_P(Geometry), _u64]
_lib.infmoe_lower_bound.restype = _f64
_lib.infmoe_lower_bound.argtypes = [_vp, _i32, _f64]
_lib.infmoe_dispatch_workspace_bytes.restype = C.c_size_t
_lib.infmoe_dispatch_workspace_bytes.argtypes = [C.c_int64, _i32]
_lib.infmoe_gaussian_fill.argtypes = [_u64, _vp, _u64]
_lib.infmoe_gaussian_fill_typed.argtypes = [_i32, _i32, _vp, _vp, _u64, _vp, _i32]
_lib.infmoe_gating_projection.argtypes = [_u64, _i32, _i32, _vp]
_lib.infmoe_lsh_codes.argtypes = [_u64, _i32, _i32, _vp, _u64, _vp]
_lib.infmoe_route_tokens.argtypes = [_u64, _i32, _i32, _vp, _u64, _i32, _vp]
_lib.infmoe_explicit_workload.argtypes = [_vp, _i32, _vp]
_lib.infmoe_workload_from_csv.argtypes = [C.c_char_p, _vp, _i32, _vp, _vp]
_lib.infmoe_simulate_orders.argtypes = [_i32, _vp, _vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp]
_lib.infmoe_synthetic_workload.argtypes = [_i32, _u64, _i32, _u64, _f64, _vp]
_lib.infmoe_compute_costs.argtypes = [_P(Geometry), _P(Hardware), _vp, _i32, _vp, _vp]
_lib.infmoe_check_constraints.argtypes = [_vp, _vp, _i32, _f64, _i32, _vp,
                                          _P(_ConstraintReport)]
_lib.infmoe_schedule.argtypes = [_vp, _i32, _f64, _i32, _i32, _i32, _vp, _vp,
                                 _P(_ScheduleInfo)]
_lib.infmoe_diagnose.argtypes = [_vp, _i32, _f64, _i32, _i32, _vp]
_lib.infmoe_simulate.argtypes = [_vp, _vp, _i32, _f64, _i32, _i32, _vp, _P(_SimReport)]
_lib.infmoe_simulate_model.argtypes = [_i32, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32,
                                       _vp, _vp, _P(_SimReport), _vp]
_lib.infmoe_fill_uniform.argtypes = [_vp, _i32, _u64, _u64, C.c_float, _vp]
_lib.infmoe_debug_occupy_sms.argtypes = [_i32, _i32, _vp, _u64, _vp, _vp]
_lib.infmoe_debug_set_flag.argtypes = [_vp, _vp]
_lib.infmoe_gate_softmax_topk.argtypes = [_vp, _i32, C.c_int64, _i32, _vp, _vp, _i32, _i32,
                                          _vp, _vp, _vp, _vp]
_lib.infmoe_layer_pack_source.argtypes = [_vp, _vp]
_lib.infmoe_set_pack_cache_dir.argtypes = [C.c_char_p]
_lib.infmoe_gate_softmax_ws_bytes.argtypes = [_i32, C.c_int64, _i32, _i32, _i32]
_lib.infmoe_gate_softmax_ws_bytes.restype = C.c_size_t
_lib.infmoe_gate_softmax_prepare.argtypes = [_vp, _i32, _i32, _vp, C.c_size_t, _vp]
_lib.infmoe_gate_softmax_topk_ws.argtypes = [_vp, _i32, C.c_int64, _i32, _vp, _vp, _i32, _i32,
                                             _vp, _vp, _vp, _vp, C.c_size_t, _vp]
_lib.infmoe_gate_softmax_debug.argtypes = [_vp, _i32, C.c_int64, _i32, _vp, _vp, _i32, _i32,
                                           _vp, _vp, _vp, _vp, _vp, _vp]
_lib.infmoe_gate_lsh.argtypes = [_vp, _i32, C.c_int64, _i32, _vp, _i32, _i32, _vp, _vp, _vp,
                                 _vp, _vp]
_lib.infmoe_dispatch.argtypes = [_vp, C.c_int64, _i32, _i32, _vp, _vp, _vp, _vp, _vp]
_lib.infmoe_gather_rows.argtypes = [_vp, _i32, C.c_int64, _i32, _i32, _vp, _vp, _vp]
_lib.infmoe_gather_rows_by_token.argtypes = [_vp, _i32, C.c_int64, _i32, _i32, _vp, _vp, _vp]
_lib.infmoe_expert_ffn.argtypes = [_vp, C.c_int64, _i32, _i32, _i32, _vp, _i32, _vp, _vp, _i32,
                                   _vp, _vp, _i32, _vp, _vp, _vp]
_lib.infmoe_combine.argtypes = [_vp, _i32, _vp, _vp, C.c_int64, _i32, _i32, _vp, _vp]
_lib.infmoe_replay_check.argtypes = [_vp, _i32, _i32, _vp, _vp, _vp, _i32, _i32, _f64, _vp,
                                     _vp]
_lib.infmoe_expert_ffn_fused.argtypes = [_vp, C.c_int64, _i32, _i32, _vp, _i32, _vp, _vp, _i32,
                                         _vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.infmoe_scatter_rows.argtypes = [_vp, _i32, C.c_int64, _i32, _vp, _vp, _vp]
_lib.infmoe_ep_plan.argtypes = [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]
_lib.infmoe_ep_get_unique_id.argtypes = [_vp]
_lib.infmoe_ep_comm_init.argtypes = [_vp, _i32, _i32, _P(_vp)]
_lib.infmoe_ep_comm_destroy.argtypes = [_vp]
_lib.infmoe_layer_create.argtypes = [_P(LayerDesc), _P(_vp)]
_lib.infmoe_layer_forward.argtypes = [_vp, _vp, C.c_int64, _vp, _P(ForwardOut), _vp]
_lib.infmoe_layer_forward_routed.argtypes = [_vp, _vp, C.c_int64, _vp, _vp, _vp,
                                             _P(ForwardOut), _vp]
_lib.infmoe_layer_set_host_weights.argtypes = [_vp, _vp, _vp]
_lib.infmoe_layer_pin_experts.argtypes = [_vp, _vp, _i32]
_lib.infmoe_layer_pin_hottest.argtypes = [_vp, _i32, _vp]
_lib.infmoe_layer_destroy.argtypes = [_vp]
_lib.infmoe_codec_roundtrip.argtypes = [_i32, _vp, _u64, _vp, _vp, _i32]
_lib.infmoe_codec_roundtrip_host.argtypes = [_i32, _vp, _u64, _vp, _vp]


def codec_roundtrip_host(bits, codec: str = "exph"):
    """Pack bf16 bit patterns with codec ("exp4" / "exph") and decode them with
    the host reference decoder (no GPU): (decoded, pack bytes)."""
    a = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty_like(a)
    nb = C.c_uint64(0)
    _check(_lib.infmoe_codec_roundtrip_host({"exp4": 1, "exph": 2}[codec],
                                            a.ctypes.data_as(_vp), a.size,
                                            out.ctypes.data_as(_vp), C.byref(nb)))
    return out, nb.value
_lib.infmoe_layer_h2d_bytes.argtypes = [_vp, _vp, _vp]
_lib.infmoe_slot_pool_create.argtypes = [_i32, _i32, _u64, _P(_vp)]
_lib.infmoe_slot_pool_create_ex.argtypes = [_i32, _i32, _u64, _i32, _P(_vp)]
_lib.infmoe_layer_set_next.argtypes = [_vp, _vp]
_lib.infmoe_slot_pool_destroy.argtypes = [_vp]


def _f64arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


# --------------------------------------------------- model_config / prng --


def geometry_preset(name: str) -> Geometry:
    g = Geometry()
    _check(_lib.infmoe_geometry_preset(name.encode(), C.byref(g)))
    return g


def make_geometry(d_model, d_ff, n_experts, bytes_per_param, n_layers=1, n_heads=1,
                  d_head=None) -> Geometry:
    return Geometry(n_layers, n_heads, d_model if d_head is None else d_head, d_model, d_ff,
                    n_experts, bytes_per_param)


def validate_geometry(g: Geometry) -> List[str]:
    w = _i32(0)
    _check(_lib.infmoe_validate_geometry(C.byref(g), C.byref(w)))
    return [f"geometry: d_model ({g.d_model}) != n_heads * d_head ({g.n_heads * g.d_head})"] \
        if w.value else []


def validate_hardware(hw: Hardware) -> None:
    _check(_lib.infmoe_validate_hardware(C.byref(hw)))


def expert_param_bytes(g: Geometry) -> int:
    return int(_lib.infmoe_expert_param_bytes(C.byref(g)))


def expert_flops(g: Geometry, n_tokens: int) -> int:
    return int(_lib.infmoe_expert_flops(C.byref(g), n_tokens))


def splitmix64(x: int) -> int:
    return int(_lib.infmoe_splitmix64(x))


def derive_seed(seed: int, tag: int) -> int:
    return int(_lib.infmoe_derive_seed(seed, tag))


def gaussian_stream(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _check(_lib.infmoe_gaussian_fill(seed, _ptr(out), n))
    return out


def gaussian_fill_typed(dtype: str, seeds, scales, n_each: int, outs, threads: int = 0) -> None:
    """SURVEY 8(d) synthetic tensors: outs[m][i] = round_dtype(GaussianStream(seeds[m])_i *
    scales[m]) (prng.hpp:49-71).  outs: host numpy arrays or raw addresses (ints, e.g. the
    data_ptr() of pinned torch tensors) of n_each elements each."""
    sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    sc = np.ascontiguousarray(np.asarray(scales, dtype=np.float64))
    if sd.size != sc.size or sd.size != len(outs):
        raise ValueError("seeds, scales and outs must have one entry per matrix")
    addr = np.array([o if isinstance(o, int) else o.ctypes.data for o in outs], dtype=np.uint64)
    code = {"bf16": DTYPE_BF16, "f32": DTYPE_F32}[dtype]
    _check(_lib.infmoe_gaussian_fill_typed(code, sd.size, _ptr(sd), _ptr(sc), n_each,
                                           _ptr(addr), threads))


def set_pack_cache_dir(path) -> None:
    """Process-wide directory of h2d-codec packs (infmoe_set_pack_cache_dir);
    None disables.  Codec layers read their pack from it instead of encoding
    when a file for the same host-weight content exists, and write it after
    encoding."""
    _check(_lib.infmoe_set_pack_cache_dir(None if path is None else str(path).encode()))


def gaussian_bf16(seed: int, n: int, scale: float = 1.0) -> np.ndarray:
    """uint16 bf16 bits of GaussianStream(seed) x scale (gaussian_tokens, gating.hpp:108-114)."""
    out = np.empty(n, dtype=np.uint16)
    gaussian_fill_typed("bf16", [seed], [scale], n, [out])
    return out


def gating_projection(seed: int, n_hash_bits: int, hidden_dim: int) -> np.ndarray:
    out = np.empty(max(n_hash_bits, 0) * max(hidden_dim, 0), dtype=np.float64)
    _check(_lib.infmoe_gating_projection(seed, n_hash_bits, hidden_dim, _ptr(out)))
    return out.reshape(n_hash_bits, hidden_dim)


def lsh_codes(seed: int, n_hash_bits: int, hidden_dim: int, hidden_states) -> np.ndarray:
    """lsh_codes (gating.hpp:61-82) on host fp64 rows [n_tokens, hidden_dim]: bit-exact."""
    x = np.ascontiguousarray(np.asarray(hidden_states, dtype=np.float64))
    n = x.size // max(hidden_dim, 1)
    if x.size != n * hidden_dim:
        raise InvalidArgument("lsh_codes: hidden_states size != n_tokens * hidden_dim")
    codes = np.zeros(n, dtype=np.uint32)
    _check(_lib.infmoe_lsh_codes(seed, n_hash_bits, hidden_dim, _ptr(x), n, _ptr(codes)))
    return codes


def route_tokens(seed: int, n_hash_bits: int, hidden_dim: int, hidden_states,
                 n_experts: int) -> np.ndarray:
    """route_tokens (gating.hpp:87-104): per-expert counts of code mod n_experts."""
    x = np.ascontiguousarray(np.asarray(hidden_states, dtype=np.float64))
    n = x.size // max(hidden_dim, 1)
    if x.size != n * hidden_dim:
        raise InvalidArgument("lsh_codes: hidden_states size != n_tokens * hidden_dim")
    counts = np.zeros(max(n_experts, 1), dtype=np.uint64)
    _check(_lib.infmoe_route_tokens(seed, n_hash_bits, hidden_dim, _ptr(x), n, n_experts,
                                    _ptr(counts)))
    return counts


def explicit_workload(counts) -> tuple:
    """explicit_workload (gating.hpp:167-175): (counts, total); ConfigError when empty."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    total = C.c_uint64(0)
    _check(_lib.infmoe_explicit_workload(_ptr(c) if c.size else None, c.size, C.byref(total)))
    return c, int(total.value)


def workload_from_csv(path) -> tuple:
    """workload_from_csv (gating.hpp:180-219): (counts, total)."""
    n = C.c_int32(0)
    total = C.c_uint64(0)
    p = str(path).encode()
    _check(_lib.infmoe_workload_from_csv(p, None, 0, C.byref(n), C.byref(total)))
    c = np.zeros(n.value, dtype=np.uint64)
    _check(_lib.infmoe_workload_from_csv(p, _ptr(c), n.value, C.byref(n), C.byref(total)))
    return c, int(total.value)


WORKLOAD_KINDS = {"uniform": 0, "zipf": 1, "balanced": 2}


def synthetic_workload(kind: str, total_tokens: int, n_experts: int, seed: int = 0,
                       zipf_s: float = 1.0) -> np.ndarray:
    if kind not in WORKLOAD_KINDS:
        raise ConfigError(f"workload.kind: unknown kind '{kind}'")
    out = np.zeros(max(n_experts, 1), dtype=np.uint64)
    _check(_lib.infmoe_synthetic_workload(WORKLOAD_KINDS[kind], total_tokens, n_experts, seed,
                                          zipf_s, _ptr(out)))
    return out


# ------------------------------------------------------------ cost model --


@dataclass
class CostVector:
    """moesim::CostVector (cost_model.hpp:22-31)."""
    alphas: np.ndarray
    beta: float

    def size(self) -> int:
        return len(self.alphas)

    def total_alpha(self) -> float:
        s = 0.0
        for a in self.alphas:
            s += float(a)
        return s


def compute_costs(counts: Sequence[int], g: Geometry, hw: Hardware) -> CostVector:
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    alphas = np.empty(len(c), dtype=np.float64)
    beta = _f64(0.0)
    _check(_lib.infmoe_compute_costs(C.byref(g), C.byref(hw), _ptr(c), len(c), _ptr(alphas),
                                     C.byref(beta)))
    return CostVector(alphas, beta.value)


def resident_capacity(g: Geometry, hw: Hardware) -> int:
    k = _i32(0)
    _check(_lib.infmoe_resident_capacity(C.byref(g), C.byref(hw), C.byref(k)))
    return k.value


def clamp_explicit_capacity(explicit_k: int, capacity: int, warnings: list) -> int:
    k, cl = _i32(0), _i32(0)
    _check(_lib.infmoe_clamp_explicit_capacity(explicit_k, capacity, C.byref(k), C.byref(cl)))
    if cl.value:
        warnings.append(f"K clamped from {explicit_k} to capacity {capacity}")
    return k.value


def with_event_overhead(c: CostVector, eps: float) -> CostVector:
    a = _f64arr(c.alphas).copy()
    b = _f64(c.beta)
    _check(_lib.infmoe_with_event_overhead(_ptr(a), len(a), C.byref(b), eps))
    return CostVector(a, b.value)


# ------------------------------------------------------------- scheduler --


@dataclass
class ConstraintReport:
    feasible: bool
    slack: np.ndarray
    first_violation: Optional[dict]


@dataclass
class Schedule:
    """moesim::Schedule (scheduler.hpp:39-45)."""
    order: List[int]
    feasible: bool
    slack: np.ndarray
    diagnosis: Optional[str]
    method: str


def check_constraints(order: Sequence[int], c: CostVector, K: int) -> ConstraintReport:
    o, a = _i32arr(order), _f64arr(c.alphas)
    slack = np.empty(max(len(a), 1), dtype=np.float64)
    rep = _ConstraintReport()
    if len(o) != len(a):
        raise ValueError(f"order size {len(o)} != expert count {len(a)}")
    _check(_lib.infmoe_check_constraints(_ptr(o), _ptr(a), len(a), c.beta, K, _ptr(slack),
                                         C.byref(rep)))
    fv = None
    if not rep.feasible:
        fv = {"position": rep.position, "bound": "lower" if rep.bound == 0 else "upper",
              "prefix_sum": rep.prefix_sum, "limit": rep.limit}
    return ConstraintReport(bool(rep.feasible), slack[:len(a)], fv)


def _schedule(c: CostVector, K: int, policy: int, max_T: int = 12) -> Schedule:
    a = _f64arr(c.alphas)
    order = np.empty(max(len(a), 1), dtype=np.int32)
    slack = np.empty(max(len(a), 1), dtype=np.float64)
    info = _ScheduleInfo()
    _check(_lib.infmoe_schedule(_ptr(a), len(a), c.beta, K, policy, max_T, _ptr(order),
                                _ptr(slack), C.byref(info)))
    return Schedule(order[:len(a)].tolist(), bool(info.feasible), slack[:len(a)],
                    DIAG[info.diagnosis], METHOD[info.method])


def greedy_order(c: CostVector, K: int) -> Schedule:
    return _schedule(c, K, POLICY_GREEDY)


def exact_order(c: CostVector, K: int, max_T: int = 12) -> Schedule:
    return _schedule(c, K, POLICY_EXACT, max_T)


def auto_order(c: CostVector, K: int, exact_fallback_max_T: int = 12) -> Schedule:
    return _schedule(c, K, POLICY_AUTO, exact_fallback_max_T)


def naive_order(c: CostVector, K: int) -> Schedule:
    return _schedule(c, K, POLICY_NAIVE)


def diagnose(c: CostVector, K: int, exact_fallback_max_T: int = 12) -> str:
    a = _f64arr(c.alphas)
    d = _i32(0)
    _check(_lib.infmoe_diagnose(_ptr(a), len(a), c.beta, K, exact_fallback_max_T, C.byref(d)))
    return DIAG[d.value]


# ------------------------------------------------------------- simulator --


@dataclass
class SimReport:
    makespan: float
    compute_busy: float
    load_busy: float
    compute_stall: float
    peak_resident_experts: int
    overlap_efficiency: float
    per_layer: list = field(default_factory=list)


def _events_list(buf, n) -> list:
    return [(buf[i].stream, buf[i].layer_id, buf[i].expert_id, buf[i].start, buf[i].end)
            for i in range(n)]


def simulate(order: Sequence[int], c: CostVector, K: int, mode: str = "overlapped"):
    """simulate(order, costs, K, mode) (simulator.hpp:209-220) -> (events, SimReport)."""
    o, a = _i32arr(order), _f64arr(c.alphas)
    if len(o) != len(a):
        raise ValueError(f"order size {len(o)} != expert count {len(a)}")
    ev = (Event * max(2 * len(a), 1))()
    rep = _SimReport()
    _check(_lib.infmoe_simulate(_ptr(o), _ptr(a), len(a), c.beta, K,
                                0 if mode == "overlapped" else 1, ev, C.byref(rep)))
    return _events_list(ev, 2 * len(a)), SimReport(rep.makespan, rep.compute_busy, rep.load_busy,
                                                    rep.compute_stall, rep.peak_resident_experts,
                                                    rep.overlap_efficiency)


def simulate_model(layer_costs: Sequence[CostVector], K: int, mode: str = "overlapped",
                   policy: str = "greedy", continuous_load_stream: bool = False,
                   exact_max_T: int = 12):
    """simulate_model(costs, K, opt) (simulator.hpp:241-255) -> (events, SimReport, orders)."""
    Ts = _i32arr([cv.size() for cv in layer_costs])
    alphas = _f64arr(np.concatenate([_f64arr(cv.alphas) for cv in layer_costs]))
    betas = _f64arr([cv.beta for cv in layer_costs])
    total = int(Ts.sum())
    orders = np.empty(max(total, 1), dtype=np.int32)
    ev = (Event * max(2 * total, 1))()
    rep = _SimReport()
    per = (_LayerReport * max(len(Ts), 1))()
    pol = {"greedy": POLICY_AUTO, "naive": POLICY_NAIVE, "exact": POLICY_EXACT}[policy]
    _check(_lib.infmoe_simulate_model(len(Ts), _ptr(Ts), _ptr(alphas), _ptr(betas), K,
                                      0 if mode == "overlapped" else 1, pol,
                                      int(continuous_load_stream), exact_max_T, _ptr(orders), ev,
                                      C.byref(rep), per))
    layers = [dict(layer_id=p.layer_id, n_experts=p.n_experts, start=p.start, end=p.end,
                   compute_busy=p.compute_busy, load_busy=p.load_busy,
                   compute_stall=p.compute_stall, peak_resident=p.peak_resident,
                   lower_bound=p.lower_bound) for p in per[:len(Ts)]]
    out_orders, off = [], 0
    for t in Ts:
        out_orders.append(orders[off:off + t].tolist())
        off += int(t)
    return (_events_list(ev, 2 * total),
            SimReport(rep.makespan, rep.compute_busy, rep.load_busy, rep.compute_stall,
                      rep.peak_resident_experts, rep.overlap_efficiency, layers), out_orders)


VIOLATION_KINDS = ("stream_overlap", "causality", "residency_exceeded", "duration_mismatch",
                   "makespan_mismatch", "malformed_event")


def replay_check(events, layer_costs: Sequence[CostVector], max_resident: int,
                 check_durations: bool = True, tol_s: float = 0.0) -> dict:
    """Audit a (simulated or measured) timeline with the rules of replay_check
    (verification.hpp:108-198).  events: (stream, layer, expert, start, end).
    Returns {kind: count} for the kinds that occurred."""
    ev = (Event * max(len(events), 1))()
    for i, (st, l, e, a, b) in enumerate(events):
        ev[i] = Event(st, l, e, a, b)
    Ts = _i32arr([cv.size() for cv in layer_costs])
    al = _f64arr(np.concatenate([_f64arr(cv.alphas) for cv in layer_costs]))
    be = _f64arr([cv.beta for cv in layer_costs])
    n = C.c_int32(0)
    kinds = np.zeros(6, np.int32)
    _check(_lib.infmoe_replay_check(ev, len(events), len(Ts), _ptr(Ts), _ptr(al), _ptr(be),
                                    max_resident, int(check_durations), tol_s, C.byref(n),
                                    _ptr(kinds)))
    return {k: int(v) for k, v in zip(VIOLATION_KINDS, kinds) if v}


def lower_bound(c: CostVector) -> float:
    a = _f64arr(c.alphas)
    return float(_lib.infmoe_lower_bound(_ptr(a), len(a), c.beta))


# ------------------------------------------------------ expert parallelism --


@dataclass
class EpPlan:
    """Exchange plan of one EP rank (csrc/host/ep_plan.cpp)."""
    send_off: np.ndarray
    send_rows: np.ndarray
    recv_off: np.ndarray
    recv_rows: np.ndarray
    local_offsets: np.ndarray
    local_index: np.ndarray
    n_recv: int


def ep_plan(P: int, rank: int, E: int, send_counts, recv_counts) -> EpPlan:
    sc = _i32arr(send_counts)
    rc = _i32arr(recv_counts).reshape(-1)
    if len(sc) != E or len(rc) != E:
        raise ValueError("ep_plan: send_counts needs E entries, recv_counts P * E/P")
    so, sr, ro, rr = (np.zeros(P, np.int64) for _ in range(4))
    lo = np.zeros(E // max(P, 1) + 1, np.int32)
    n = C.c_int64(0)
    _check(_lib.infmoe_ep_plan(P, rank, E, _ptr(sc), _ptr(rc), _ptr(so), _ptr(sr), _ptr(ro),
                               _ptr(rr), _ptr(lo), None, C.byref(n)))
    li = np.zeros(max(n.value, 1), np.int32)
    _check(_lib.infmoe_ep_plan(P, rank, E, _ptr(sc), _ptr(rc), None, None, None, None, None,
                               _ptr(li), None))
    return EpPlan(so, sr, ro, rr, lo, li[:n.value], n.value)


def ep_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.infmoe_ep_get_unique_id(buf))
    return bytes(buf)


def ep_comm_init(uid: bytes, nranks: int, rank: int) -> int:
    buf = (C.c_uint8 * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    _check(_lib.infmoe_ep_comm_init(buf, nranks, rank, C.byref(comm)))
    return comm.value


def ep_comm_destroy(comm: int) -> None:
    _check(_lib.infmoe_ep_comm_destroy(C.c_void_p(comm)))


from . import device  # noqa: E402,F401  (device-path wrappers over torch tensors)
