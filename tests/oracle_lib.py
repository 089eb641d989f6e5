"""ctypes access to the CHECKERS (test infrastructure only).

- ``O``   : oracle/liboracle.so — the CPU restatement (oracle/oracle.c)
- ``REF`` : oracle/_ref/libmoesim_ref.so — the reference headers compiled in
            place (None when neither /root/reference nor a prebuilt copy exists)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"


def _ensure_built() -> None:
    so = ORACLE_DIR / "liboracle.so"
    ref = ORACLE_DIR / "_ref" / "libmoesim_ref.so"
    need = (not so.exists()) or so.stat().st_mtime < (ORACLE_DIR / "oracle.c").stat().st_mtime
    need = need or (not ref.exists() and Path("/root/reference/proj/include").exists())
    if need:
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)


_ensure_built()
O = C.CDLL(str(ORACLE_DIR / "liboracle.so"))
_ref_path = ORACLE_DIR / "_ref" / "libmoesim_ref.so"
REF = C.CDLL(str(_ref_path)) if _ref_path.exists() else None

u64, i32, f64, vp = C.c_uint64, C.c_int32, C.c_double, C.c_void_p

for lib, pre in ((O, "or_"), (REF, "ref_")):
    if lib is None:
        continue
    for name in ("splitmix64", "mt64_first"):
        fn = getattr(lib, pre + name, None)
        if fn is not None:
            fn.restype = u64
            fn.argtypes = [u64]
    getattr(lib, pre + "derive_seed").restype = u64
    getattr(lib, pre + "derive_seed").argtypes = [u64, u64]
    getattr(lib, pre + "expert_param_bytes").restype = u64
    getattr(lib, pre + "expert_flops").restype = u64
    getattr(lib, pre + "expert_flops").argtypes = [C.c_int, C.c_int, u64]
    getattr(lib, pre + "instance_digest").restype = u64
    getattr(lib, pre + "instance_digest").argtypes = [vp, C.c_int, f64, C.c_int]
    getattr(lib, pre + "lower_bound").restype = f64
    getattr(lib, pre + "lower_bound").argtypes = [vp, C.c_int, f64]
    getattr(lib, pre + "compute_costs").argtypes = [C.c_int, C.c_int, C.c_int, f64, f64, vp,
                                                   C.c_int, vp, vp]
    getattr(lib, pre + "resident_capacity").argtypes = [C.c_int, C.c_int, C.c_int, u64, u64, vp]
    getattr(lib, pre + "check_constraints").argtypes = [vp, vp, C.c_int, f64, C.c_int, vp, vp,
                                                       vp, vp]
    getattr(lib, pre + "diagnose").argtypes = [vp, C.c_int, f64, C.c_int, C.c_int]
    getattr(lib, pre + "enumerate_feasibility").argtypes = [vp, C.c_int, f64, C.c_int, vp]
    getattr(lib, pre + "synthetic_workload").argtypes = [C.c_int, u64, C.c_int, u64, f64, vp]
    getattr(lib, pre + "gating_projection").argtypes = [u64, C.c_int, C.c_int, vp]
    getattr(lib, pre + "lsh_codes").argtypes = [u64, C.c_int, C.c_int, vp, u64, vp]
    getattr(lib, pre + "route_tokens").argtypes = [u64, C.c_int, C.c_int, vp, u64, C.c_int, vp]

O.or_gaussian_fill.argtypes = [u64, vp, u64]
O.or_fill_uniform_f32.argtypes = [u64, u64, C.c_float, vp]
O.or_fill_uniform_bf16.argtypes = [u64, u64, C.c_float, vp]
O.or_greedy_order.argtypes = [vp, C.c_int, f64, C.c_int, vp, vp, vp]
O.or_exact_order.argtypes = [vp, C.c_int, f64, C.c_int, C.c_int, vp, vp, vp]
O.or_auto_order.argtypes = [vp, C.c_int, f64, C.c_int, C.c_int, vp, vp, vp, vp]
O.or_run_layers.argtypes = [C.c_int, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]
O.or_replay_check.argtypes = [vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, C.c_int, vp]
O.or_gate_softmax.argtypes = [vp, u64, C.c_int, vp, vp, C.c_int, C.c_int, vp, vp, vp]
O.or_gate_lsh.argtypes = [vp, u64, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp]
O.or_dispatch.argtypes = [vp, u64, C.c_int, C.c_int, vp, vp, vp]
O.or_expert_ffn.argtypes = [vp, u64, C.c_int, C.c_int, vp, vp, C.c_int, vp]
O.or_combine.argtypes = [vp, vp, vp, u64, C.c_int, C.c_int, vp]
if REF is not None:
    REF.ref_gaussian_tokens.argtypes = [u64, u64, C.c_int, vp]
    REF.ref_schedule.argtypes = [vp, C.c_int, f64, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp]
    REF.ref_simulate_model.argtypes = [C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, vp, vp, vp]
    REF.ref_simulate_order.argtypes = [vp, vp, C.c_int, f64, C.c_int, C.c_int, vp, vp]
    REF.ref_replay_check.argtypes = [vp, C.c_int, vp, C.c_int, f64, C.c_int, vp]


class EventRec(C.Structure):
    _fields_ = [("stream", C.c_int), ("layer_id", C.c_int), ("expert_id", C.c_int),
                ("start", C.c_double), ("end", C.c_double)]


class ReportRec(C.Structure):
    _fields_ = [("makespan", C.c_double), ("compute_busy", C.c_double),
                ("load_busy", C.c_double), ("compute_stall", C.c_double),
                ("peak_resident", C.c_int), ("overlap_efficiency", C.c_double)]


def ptr(a: np.ndarray):
    return a.ctypes.data_as(vp)


def f64a(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def i32a(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


# ---------------------------------------------------------------- helpers --


def gaussian(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    O.or_gaussian_fill(seed, ptr(out), n)
    return out


def fill_bf16(seed: int, n: int, scale: float) -> np.ndarray:
    """uint16 bf16 bits of the counter-hash fill."""
    out = np.empty(n, dtype=np.uint16)
    O.or_fill_uniform_bf16(seed, n, scale, ptr(out))
    return out


def fill_f32(seed: int, n: int, scale: float) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    O.or_fill_uniform_f32(seed, n, scale, ptr(out))
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def schedule(lib_prefix: str, alphas, beta: float, K: int, policy: str, max_T: int = 12):
    """policy: auto | greedy | exact | naive.  Returns (order, feasible, diagnosis, method)."""
    a = f64a(alphas)
    T = len(a)
    order = np.zeros(T, dtype=np.int32)
    feas, diag, meth = C.c_int(0), C.c_int(0), C.c_int(0)
    if lib_prefix == "ref":
        pol = {"auto": 0, "greedy": 1, "exact": 2, "naive": 3}[policy]
        rc = REF.ref_schedule(ptr(a), T, beta, K, pol, max_T, ptr(order), C.byref(feas),
                              C.byref(diag), C.byref(meth))
    else:
        if policy == "greedy":
            rc = O.or_greedy_order(ptr(a), T, beta, K, ptr(order), C.byref(feas), C.byref(diag))
        elif policy == "exact":
            rc = O.or_exact_order(ptr(a), T, beta, K, max_T, ptr(order), C.byref(feas),
                                  C.byref(diag))
            meth.value = 1
        elif policy == "auto":
            rc = O.or_auto_order(ptr(a), T, beta, K, max_T, ptr(order), C.byref(feas),
                                 C.byref(diag), C.byref(meth))
        else:
            raise ValueError(policy)
    return rc, order.tolist(), bool(feas.value), diag.value, meth.value
