"""cpu_stack.py — the CPU path of the MoE stack (TEST / BASELINE INFRASTRUCTURE:
only bench.py's cpu_baseline leg and `bench.py --impl reference` use it; the
product never imports anything under oracle/).

One forward pass of the offloaded-stack workload on the host cores, through the
REFERENCE's own code wherever the reference has any -- oracle/_ref is the
moesim headers compiled in place, unmodified (oracle/Makefile):

* inputs   gaussian_tokens / GaussianStream        (gating.hpp:108-114, prng.hpp:49-71)
* gate     gating_projection + lsh_codes, expert = code mod E  (gating.hpp:38-104)
* schedule compute_costs + auto_order per layer    (cost_model.hpp:43-62, scheduler.hpp:243)

and through the oracle PORT for the pieces the reference lacks:
dispatch (oracle.c or_dispatch), the expert FFN over bf16 weights read in place
with fp32 accumulation (cpu_ffn.c or_expert_ffn_bf16, AVX512-BF16 where the host
has it, OpenMP over all cores) and the top-1 combine (y = bf16(w * bf16(acc)),
w = 1 for the LSH gate).  On the CPU the weights are read where they live, so
the InfMoE order only fixes the order the experts are computed in.
"""
from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import os
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
vp, u64, i32, f64 = C.c_void_p, C.c_uint64, C.c_int, C.c_double


def _load():
    lib = C.CDLL(str(HERE / "liboracle.so"))
    lib.or_dispatch.argtypes = [vp, u64, i32, i32, vp, vp, vp]
    lib.or_expert_ffn_bf16.argtypes = [vp, u64, i32, i32, vp, vp, vp, vp]
    lib.or_cpu_ffn_isa.restype = i32
    ref_so = HERE / "_ref" / "libmoesim_ref.so"
    ref = C.CDLL(str(ref_so)) if ref_so.exists() else None
    if ref is not None:
        ref.ref_derive_seed.restype = u64
        ref.ref_derive_seed.argtypes = [u64, u64]
        ref.ref_gaussian_tokens.argtypes = [u64, u64, i32, vp]
        ref.ref_gating_projection.argtypes = [u64, i32, i32, vp]
        ref.ref_lsh_codes.argtypes = [u64, i32, i32, vp, u64, vp]
        ref.ref_compute_costs.argtypes = [i32, i32, i32, f64, f64, vp, i32, vp, vp]
        ref.ref_schedule.argtypes = [vp, i32, f64, i32, i32, i32, vp, vp, vp, vp]
    return lib, ref


O, REF = _load()


def P(a: np.ndarray):
    return a.ctypes.data_as(vp)


def f64_to_bf16_bits(v: np.ndarray) -> np.ndarray:
    """double -> f32 (RN) -> bf16 (RNE): the rounding of the GPU arm's inputs."""
    u = np.ascontiguousarray(v.astype(np.float32)).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def bf16_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


class Derive:
    """derive_seed through the reference build (prng.hpp:27-29)."""

    @staticmethod
    def derive_seed(seed: int, tag: int) -> int:
        return int(REF.ref_derive_seed(seed, tag))


def ref_gaussian_bf16(seed: int, n: int, scale: float) -> np.ndarray:
    """GaussianStream(seed) x scale, rounded to bf16, through oracle/_ref."""
    g = np.empty(n, np.float64)
    REF.ref_gaussian_tokens(seed, n, 1, P(g))
    return f64_to_bf16_bits(g * scale)


def ref_expert_weights(scen_seed: int, e0: int, n: int, d: int, f: int, threads: int):
    """The GPU arm's expert weights (bench.py fill_expert_weights) via oracle/_ref:
    W_in[e] = GaussianStream(derive_seed(S, 1000+2e)) x d^-1/2, W_out[e] = ... 1001+2e
    x f^-1/2, bf16.  Returns (w_in [n, f, d], w_out [n, d, f]) uint16."""
    wi = np.empty((n, f, d), np.uint16)
    wo = np.empty((n, d, f), np.uint16)
    jobs = [(wi, e, Derive.derive_seed(scen_seed, 1000 + 2 * (e0 + e)), d ** -0.5)
            for e in range(n)] + \
           [(wo, e, Derive.derive_seed(scen_seed, 1001 + 2 * (e0 + e)), f ** -0.5)
            for e in range(n)]

    def run(job):
        dst, e, seed, scale = job
        dst[e] = ref_gaussian_bf16(seed, f * d, scale).reshape(dst.shape[1:])

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(run, jobs))
    return wi, wo


class CpuStack:
    """A stack of offloaded MoE layers on the host: layer l uses weight set
    l % n_sets (w_sets[s] = (w_in [E, f, d], w_out [E, d, f]) bf16 bits) and the
    LSH gate GatingModel{lsh_seeds[l], bits, d}."""

    def __init__(self, d, f, E, bits, K, lsh_seeds, w_sets, peak_flops, h2d_bw):
        self.d, self.f, self.E, self.bits, self.K = d, f, E, bits, K
        self.lsh_seeds = list(lsh_seeds)
        self.w_sets = w_sets
        self.peak_flops, self.h2d_bw = peak_flops, h2d_bw
        self.isa = "avx512_bf16 vdpbf16ps" if O.or_cpu_ffn_isa() else "fp32 fma (generic)"

    def layer(self, x_bits: np.ndarray, l: int, info: dict | None = None) -> np.ndarray:
        d, f, E = self.d, self.f, self.E
        n = x_bits.shape[0]
        wi, wo = self.w_sets[l % len(self.w_sets)]
        # gate: the reference's lsh_codes on the fp64 promotion of the bf16 rows
        xd = np.ascontiguousarray(bf16_to_f64(x_bits.reshape(-1)))
        codes = np.empty(n, np.uint32)
        REF.ref_lsh_codes(self.lsh_seeds[l], self.bits, d, P(xd), n, P(codes))
        idx = (codes % np.uint32(E)).astype(np.int32)
        counts = np.bincount(idx, minlength=E).astype(np.uint64)
        # InfMoE order (the reference scheduler) for these counts
        alphas = np.zeros(E, np.float64)
        beta = C.c_double(0.0)
        REF.ref_compute_costs(d, f, 2, self.peak_flops, self.h2d_bw, P(counts), E, P(alphas),
                              C.byref(beta))
        order = np.zeros(E, np.int32)
        fz = [np.zeros(1, np.int32) for _ in range(3)]
        REF.ref_schedule(P(alphas), E, beta.value, self.K, 0, 12, P(order), P(fz[0]), P(fz[1]),
                         P(fz[2]))
        # dispatch (port): stable counting sort by expert
        off = np.zeros(E + 1, np.int32)
        perm = np.zeros(n, np.int32)
        inv = np.zeros(n, np.int32)
        O.or_dispatch(P(idx), n, 1, E, P(off), P(perm), P(inv))
        xp = np.ascontiguousarray(x_bits[perm])
        yp = np.empty((n, d), np.float32)
        h = np.empty((max(int(counts.max()), 1), f), np.uint16)
        for e in order.tolist():
            a, b = int(off[e]), int(off[e + 1])
            if b > a:
                O.or_expert_ffn_bf16(P(xp[a:b]), b - a, d, f, P(wi[e]), P(wo[e]), P(h),
                                     P(yp[a:b]))
        # combine (top-1, weight 1): y[t] = bf16(1 * bf16(acc))
        y = f32_to_bf16_bits(yp)[inv]
        if info is not None:
            info.setdefault("counts", []).append(counts)
            info.setdefault("order", []).append(order)
        return y

    def forward(self, x_bits: np.ndarray, n_layers: int, info: dict | None = None) -> np.ndarray:
        cur = x_bits
        for l in range(n_layers):
            cur = self.layer(cur, l, info)
        return cur


def cpu_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical cpus)"
    except OSError:
        pass
    return f"unknown ({os.cpu_count()} logical cpus)"


def timed_passes(stack: CpuStack, x_bits, n_layers, steps, warmup):
    out, ts = None, []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        out = stack.forward(x_bits, n_layers)
        if i >= warmup:
            ts.append(time.perf_counter() - t0)
    return out, ts
