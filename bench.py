#!/usr/bin/env python
"""bench.py — InfMoE MoE-layer hot path on B200 (BASELINE.json metric).

Default workload (BASELINE.json configs[2], "C3"): the CPM-2-MoE 24-layer
decoder MoE stack, d_model 4096, d_ff 10240, 32 experts/layer, top-1 LSH gate
(the CPM-2 gate, gating.hpp:61-104), 4096 tokens, bf16, expert weights
offloaded to pinned host memory and streamed in the InfMoE load order with
K=4 resident experts per layer (K+1 device slots).  A step is one forward pass
of the 4096 tokens through all 24 MoE layers.

Reported in ONE JSON line (rank 0):
  value  tokens/s through the offloaded stack, inputs already in HBM
  e2e    the same through the C-ABI layer handles with the input copied from
         pinned host memory and the output read back inside the timed region
  h2d    achieved host-link GB/s vs the measured pinned peak, exposed copy time
  roofline  the dominant GPU kernel (the expert FFN GEMM pair) vs measured HBM
  resident  the same stack with all experts resident in HBM (C2/C4 regime)
  cpu_baseline  the oracle port of the same layer on the host cores
`--impl reference` times the CPU reference path instead.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = 20261018

CONFIGS = {
    # BASELINE.json configs[2]: the headline (metric quoted on 1 B200 offloaded)
    "c3": dict(workload="cpm2-moe-24L-decoder-stack-offloaded", d=4096, f=10240, E=32, k=1,
               N=4096, L=24, gate="lsh", bits=5, K=4),
    # configs[0] (C1, fp32 CPU-runnable) and configs[4] (C5, E64 top-2 Zipf) are
    # parity cases, not bench lines: tests/test_gpu_fullsize.py runs them at
    # full size against the oracle and the reference scheduler
}


def bind_to_gpu_numa_node(dev_index: int) -> str:
    """Multi-rank runs: restrict this process to the CPUs NVML reports as local
    to its GPU before any pinned host memory is allocated, so first-touch places
    the rank's expert weights (streamed over the GPU's own host link) on the
    near NUMA node.  A no-op on one-node hosts; never fatal."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(dev_index).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid).encode())
        n = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(n))
        if cpus and cpus != set(os.sched_getaffinity(0)):
            os.sched_setaffinity(0, cpus)
            return f"{len(cpus)} cpus near the GPU"
        return "unchanged (every cpu is near the GPU)"
    except Exception as e:  # noqa: BLE001 - affinity is an optimisation only
        return f"unchanged ({type(e).__name__})"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def lsh_seed(lib, layer: int) -> int:
    """Layer l's LSH gate: GatingModel{derive_seed(S_l, 2), bits, d} with S_l = SEED + l
    (SURVEY 8(d)); `lib` provides derive_seed (the package, or oracle/_ref in the
    reference arm -- the same splitmix64 values)."""
    return int(lib.derive_seed(SEED + layer, 2))


def fill_expert_weights(im, scen_seed: int, e0: int, n: int, d: int, f: int, hi, ho) -> None:
    """W_in[e] = GaussianStream(derive_seed(S, 1000 + 2e)) x d^-1/2 and
    W_out[e] = GaussianStream(derive_seed(S, 1001 + 2e)) x f^-1/2 for the global experts
    e0 .. e0+n-1, rounded to bf16, written into the (pinned) host tensors hi [n, f, d] and
    ho [n, d, f] on all host threads."""
    seeds = [im.derive_seed(scen_seed, 1000 + 2 * (e0 + e)) for e in range(n)] + \
            [im.derive_seed(scen_seed, 1001 + 2 * (e0 + e)) for e in range(n)]
    scales = [d ** -0.5] * n + [f ** -0.5] * n
    outs = [hi[e].data_ptr() for e in range(n)] + [ho[e].data_ptr() for e in range(n)]
    im.gaussian_fill_typed("bf16", seeds, scales, f * d, outs)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["_src"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "_src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline --

def _cpu_stack_module():
    """oracle/cpu_stack.py: the CPU path (reference code from oracle/_ref where the
    reference has any, the oracle port elsewhere).  Only the CPU legs import it."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import cpu_stack
    return cpu_stack


def layer0_parity(cfg, x_bits: np.ndarray, w_in_bits, w_out_bits, proj, y_gpu: np.ndarray,
                  counts_gpu, perm_gpu) -> dict:
    """Layer 0 of the stack on ALL its tokens against the fp64 CPU oracle (LSH gate
    -> dispatch -> fp64-accumulated FFN with H rounded to bf16 -> combine): routing
    counts and permutation bit-exact, max-abs / relative-L2 error of y.  The oracle is
    the checker here, not a timed arm."""
    lib = C.CDLL(str(ROOT / "oracle" / "liboracle.so"))
    vp = C.c_void_p
    lib.or_gate_lsh.argtypes = [vp, C.c_uint64, C.c_int, vp, C.c_int, C.c_int, vp, vp, vp]
    lib.or_dispatch.argtypes = [vp, C.c_uint64, C.c_int, C.c_int, vp, vp, vp]
    lib.or_expert_ffn.argtypes = [vp, C.c_uint64, C.c_int, C.c_int, vp, vp, C.c_int, vp]
    lib.or_combine.argtypes = [vp, vp, vp, C.c_uint64, C.c_int, C.c_int, vp]
    P = lambda a: a.ctypes.data_as(vp)
    d, f, E = cfg["d"], cfg["f"], cfg["E"]
    n = x_bits.shape[0]
    to_f32 = lambda b: (b.astype(np.uint32) << 16).view(np.float32)
    x = np.ascontiguousarray(to_f32(x_bits.reshape(-1)).reshape(n, d))
    t0 = time.perf_counter()
    idx = np.zeros((n, 1), np.int32)
    w = np.zeros((n, 1), np.float32)
    cnt = np.zeros(E, np.int32)
    lib.or_gate_lsh(P(x), n, d, P(proj), proj.shape[0], E, P(idx), P(w), P(cnt))
    off = np.zeros(E + 1, np.int32)
    perm = np.zeros(n, np.int32)
    inv = np.zeros(n, np.int32)
    lib.or_dispatch(P(idx), n, 1, E, P(off), P(perm), P(inv))
    xp = np.ascontiguousarray(x[perm])
    yp = np.zeros((n, d), np.float32)
    for e in range(E):
        a, b = int(off[e]), int(off[e + 1])
        if b > a:
            wi = np.ascontiguousarray(to_f32(w_in_bits[e].reshape(-1)))
            wo = np.ascontiguousarray(to_f32(w_out_bits[e].reshape(-1)))
            lib.or_expert_ffn(P(xp[a:b]), b - a, d, f, P(wi), P(wo), 1, P(yp[a:b]))
    # the device stores y_perm in bf16 before the combine
    yp = to_f32(((yp.view(np.uint32).astype(np.uint64) + 0x7FFF +
                  ((yp.view(np.uint32) >> 16) & 1)) >> 16).astype(np.uint16))
    y = np.zeros((n, d), np.float32)
    lib.or_combine(P(np.ascontiguousarray(yp)), P(inv), P(w), n, 1, d, P(y))
    err = np.abs(y_gpu - y)
    tol = 3e-2 + 2e-2 * np.abs(y)
    return {"tokens": int(n), "layer": 0, "oracle_seconds": time.perf_counter() - t0,
            "counts_bit_exact": bool(np.array_equal(np.asarray(counts_gpu), cnt)),
            "perm_bit_exact": bool(np.array_equal(np.asarray(perm_gpu), perm)),
            "max_abs_err": float(err.max()), "mean_abs_err": float(err.mean()),
            "rel_l2_err": float(np.linalg.norm(err) / np.linalg.norm(y)),
            "max_err_over_tol": float((err / tol).max()),
            "tolerance": "|y - y_ref| <= 3e-2 + 2e-2 |y_ref| (bf16 output)",
            "within_tolerance": bool(np.all(err <= tol))}


def reference_pieces(cfg, cs) -> dict | None:
    """Time the reference's own CPU pieces of this path as shipped (the moesim
    headers compiled in place into oracle/_ref, single thread): gaussian_tokens,
    route_tokens, compute_costs + auto_order per layer, simulate_model over the
    stack (SURVEY.md 8(d) "CPU path timed beside the GPU", item i)."""
    lib = cs.REF
    if lib is None or cfg["gate"] != "lsh":
        return None
    vp, u64 = C.c_void_p, C.c_uint64
    lib.ref_route_tokens.argtypes = [u64, C.c_int, C.c_int, vp, u64, C.c_int, vp]
    lib.ref_simulate_model.argtypes = [C.c_int, vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, vp, vp, vp]
    P = lambda a: a.ctypes.data_as(vp)
    d, E, N, L, bits, K = cfg["d"], cfg["E"], cfg["N"], cfg["L"], cfg["bits"], cfg["K"]
    out = {"impl": "oracle/_ref (reference headers, g++ -O2, 1 thread)", "cpu": cs.cpu_model(),
           "shape": f"{N} tokens x d {d}, {bits} bits, E {E}, {L} layers, K {K}"}
    x = np.empty(N * d, np.float64)
    t0 = time.perf_counter()
    lib.ref_gaussian_tokens(lib.ref_derive_seed(SEED, 0), N, d, P(x))
    out["gaussian_tokens_ms"] = (time.perf_counter() - t0) * 1e3
    route = {}
    for name, (n, dd, b, e) in {"c1_512x768_3b": (512, 768, 3, 8), "c2_4096x4096_5b": (N, d, bits, E),
                                "c5_16384x4096_6b": (16384, 4096, 6, 64)}.items():
        xs = x if (n, dd) == (N, d) else np.empty(n * dd, np.float64)
        if xs is not x:
            lib.ref_gaussian_tokens(lib.ref_derive_seed(SEED, 7), n, dd, P(xs))
        cnt = np.zeros(e, np.uint64)
        t0 = time.perf_counter()
        lib.ref_route_tokens(lsh_seed(cs.Derive, 0), b, dd, P(xs), n, e, P(cnt))
        route[name] = (time.perf_counter() - t0) * 1e3
    out["route_tokens_ms"] = route
    cnt = np.zeros(E, np.uint64)
    lib.ref_route_tokens(lsh_seed(cs.Derive, 0), bits, d, P(x), N, E, P(cnt))
    co = {}
    for T in (32, 64):
        cT = np.resize(cnt, T).astype(np.uint64)
        alphas = np.zeros(T, np.float64)
        beta = C.c_double(0.0)
        order = np.zeros(T, np.int32)
        fz = [np.zeros(1, np.int32) for _ in range(3)]
        reps = 200
        t0 = time.perf_counter()
        for _ in range(reps):
            lib.ref_compute_costs(d, cfg["f"], 2, 1643.6e12, 55.5e9, P(cT), T, P(alphas),
                                  C.byref(beta))
            lib.ref_schedule(P(alphas), T, beta.value, K, 0, 12, P(order), P(fz[0]), P(fz[1]),
                             P(fz[2]))
        co[f"T{T}"] = (time.perf_counter() - t0) / reps * 1e6
    out["costs_plus_auto_order_us"] = co
    alphas = np.zeros(E, np.float64)
    beta = C.c_double(0.0)
    lib.ref_compute_costs(d, cfg["f"], 2, 1643.6e12, 55.5e9, P(cnt), E, P(alphas), C.byref(beta))
    Ts = np.full(L, E, np.int32)
    al = np.tile(alphas, L)
    be = np.full(L, beta.value)
    orders = np.zeros(L * E, np.int32)
    ev = np.zeros(2 * L * E * 5, np.float64)  # 2 events per expert, 40 B each (>= ref_event)
    rep = np.zeros(8, np.float64)
    t0 = time.perf_counter()
    lib.ref_simulate_model(L, P(Ts), P(al), P(be), K, 0, 0, 0, 12, P(orders), P(ev), P(rep))
    out["simulate_model_ms"] = (time.perf_counter() - t0) * 1e3
    out["simulated_makespan_s"] = float(rep[0])
    return out


def repo_libs_loaded() -> list:
    """The shared objects of this repository mapped into this process."""
    try:
        maps = open("/proc/self/maps").read().splitlines()
    except OSError:
        return []
    return sorted({ln.split()[-1][len(str(ROOT)) + 1:] for ln in maps
                   if ln.split()[-1].startswith(str(ROOT)) and ".so" in ln})


def bench_config(cfg, args, P: int, n_sets: int) -> dict:
    """The `config` object of BOTH arms (the reference arm runs the same workload)."""
    return {"workload": cfg["workload"], "tokens": cfg["N"], "layers": cfg["L"],
            "d_model": cfg["d"], "d_ff": cfg["f"], "experts": cfg["E"], "top_k": cfg["k"],
            "gate": cfg["gate"], "K": cfg["K"], "device_slots": cfg["K"] + 1,
            "slot_pool": "one pool of K+1 slots shared by all layers",
            "policy": "infmoe_greedy(auto_order)", "host_weight_sets": n_sets,
            "parallelism": f"ep{P}" if P > 1 else "single",
            "ep_transport": args.ep_transport if P > 1 else None,
            "h2d_codec": args.h2d_codec,
            "inputs": "SURVEY 8(d): x = gaussian_tokens(derive_seed(S,0)); W_in/W_out[e] = "
                      "GaussianStream(derive_seed(S_s,1000+2e / 1001+2e)) x d^-1/2 / f^-1/2, "
                      "S_s = S + set; LSH gate of layer l = GatingModel{derive_seed(S+l,2)}; "
                      "S = 20261018; bf16 (f32 RN then RNE)",
            "l2": "inputs larger than L2 (5.37 GB of expert weights per layer)"}


def run_reference_arm(args, cfg, rank: int) -> None:
    """--impl reference: the CPU path of the same workload on all host cores
    (oracle/cpu_stack.py: the reference's own gaussian_tokens / GaussianStream,
    lsh_codes and compute_costs + auto_order from oracle/_ref; the oracle port for
    dispatch, the bf16 FFN with fp32 accumulation, combine).  Each step is ONE
    real pass of a token sample through all L layers; libinfmoe is never loaded."""
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    cs = _cpu_stack_module()
    if cs.REF is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the reference "
                          "headers compiled in place) is missing"}), flush=True)
        return
    d, f, E, L = cfg["d"], cfg["f"], cfg["E"], cfg["L"]
    n_tok = args.cpu_sample
    n_sets = max(1, min(args.host_sets, L))
    threads = cs.cpu_threads()
    peaks = measured_peaks()
    t0 = time.perf_counter()
    w_sets = [cs.ref_expert_weights(SEED + s, 0, E, d, f, threads) for s in range(n_sets)]
    x_bits = cs.ref_gaussian_bf16(cs.Derive.derive_seed(SEED, 0), n_tok * d, 1.0).reshape(n_tok, d)
    gen_s = time.perf_counter() - t0
    stack = cs.CpuStack(d, f, E, cfg["bits"], cfg["K"], [lsh_seed(cs.Derive, l) for l in range(L)],
                        w_sets, float(peaks["bf16_tflops"]) * 1e12, 55.6e9)
    _, ts = cs.timed_passes(stack, x_bits, L, args.steps, args.warmup)
    t_pass = float(np.mean(ts))
    value = n_tok / t_pass
    sample = (f"the first {n_tok} of the workload's {cfg['N']} tokens through all {L} layers per "
              f"step (a real {L}-layer pass; tokens are independent rows)")
    line = {"metric": "moe_stack_tokens_per_s", "value": value, "unit": "tokens/s",
            "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_pass * 1e3,
            "ms_per_step_all": [t * 1e3 for t in ts],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (SURVEY 8(d) generators through oracle/_ref; random-init weights)",
            "config": bench_config(cfg, args, 1, n_sets),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads,
                             "kind": "port", "cpu": cs.cpu_model(), "sample": sample,
                             "path": "reference code (oracle/_ref): gaussian_tokens, lsh_codes, "
                                     "compute_costs + auto_order; oracle port: dispatch, FFN "
                                     f"(bf16 in place, fp32 accumulation, {stack.isa}), combine",
                             "input_generation_s": gen_s},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    pieces = reference_pieces(cfg, cs)
    if pieces is not None:
        line["reference_pieces"] = pieces
    line["native_libs_loaded"] = repo_libs_loaded()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm --

# ------------------------------------------- C5: skewed routing, offloaded --

C5 = dict(workload="skewed-routing-stress-E64-top2-zipf-offloaded", d=4096, f=10240, E=64, k=2,
          N=16384, K=4)
C5_SEED = SEED + 500  # the C5 scenario seed


def _l2_flush(torch, dev):
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    return lambda: buf.zero_()  # 256 MB > the 126 MB L2


def measure_c5(torch, im, dv, dev, local, stream, peaks, h2d_peak, reps: int = 3) -> dict:
    """BASELINE.json configs[4] (C5) on one GPU: E=64 top-2 softmax gate skewed
    by a logit bias b_e = -ln(e+1) (Zipf-like realised loads),
    16384 tokens, offloaded with K=4 in the InfMoE order; the same layer
    resident (tensor-bound: ~512 rows per expert); and the dispatch/combine
    kernels at this size (the HBM-bound data movement of the path)."""
    c = C5
    N, d, f, E, k, K = c["N"], c["d"], c["f"], c["E"], c["k"], c["K"]
    bf = torch.bfloat16
    S5 = C5_SEED
    # SURVEY 8(d) inputs at scenario seed S5: W_in/W_out[e] from GaussianStream x
    # d^-1/2 / f^-1/2, x = gaussian_tokens(derive_seed(S5, 0)), W_g [d, E] =
    # GaussianStream(derive_seed(S5, 1)) x d^-1/2 (the layer takes it as [E, d])
    hi = torch.empty((E, f, d), dtype=bf, pin_memory=True)
    ho = torch.empty((E, d, f), dtype=bf, pin_memory=True)
    fill_expert_weights(im, S5, 0, E, d, f, hi, ho)
    wi, wo = hi.to(dev), ho.to(dev)
    xb = im.gaussian_bf16(im.derive_seed(S5, 0), N * d)
    x = torch.from_numpy(xb.view(np.int16).reshape(N, d)).view(bf).to(dev)
    gw = np.ascontiguousarray(
        (im.gaussian_stream(im.derive_seed(S5, 1), d * E) * d ** -0.5).astype(np.float32)
        .reshape(d, E).T)
    # skew: logit bias b_e = -c ln(e+1), c calibrated (bisection on the GPU gate's
    # realised counts) so the most-loaded expert matches the Zipf(1) pin of the same
    # size, synthetic_workload(Zipf, N*k, E, S5, 1.0) (gating.hpp:122-165)
    zipf = np.sort(im.synthetic_workload("zipf", N * k, E, S5, 1.0))[::-1]
    wg_dev = torch.from_numpy(gw).to(dev)
    lnr = -np.log(np.arange(1, E + 1))

    def top_counts(cc):
        b = torch.from_numpy((cc * lnr).astype(np.float32)).to(dev)
        return np.sort(dv.gate_softmax_topk(x, wg_dev, k, bias=b)[2].cpu().numpy())[::-1]

    lo, hi_c = 0.0, 8.0
    for _ in range(40):
        mid = 0.5 * (lo + hi_c)
        if top_counts(mid)[0] < zipf[0]:
            lo = mid
        else:
            hi_c = mid
    c_bias = 0.5 * (lo + hi_c)
    bias = (c_bias * lnr).astype(np.float32)
    hw = im.Hardware(float(peaks["bf16_tflops"]) * 1e12, h2d_peak * 1e9, 180 << 30, 8 << 30)
    kw = dict(gate="softmax", gate_weight=gw, gate_bias=bias, max_tokens=N, device=local, hw=hw)
    res = dv.MoELayer(d, f, E, k, wi, wo, **kw)
    off = dv.MoELayer(d, f, E, k, hi, ho, offloaded=True, K=K, **kw)
    offh = dv.MoELayer(d, f, E, k, hi, ho, offloaded=True, K=K, h2d_codec="exph", **kw)
    # the reference's skip_empty_experts option (scenario.hpp:99):
    # experts that received no rows are neither scheduled nor loaded
    off_skip = dv.MoELayer(d, f, E, k, hi, ho, offloaded=True, K=K, h2d_codec="exph",
                           skip_empty_experts=True, **kw)
    y_off, y_res = torch.empty_like(x), torch.empty_like(x)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        off.forward(x, y_off)
        res.forward(x, y_res, want_info=False)
    torch.cuda.synchronize()
    # offloaded: the host link binds (64 x 167.8 MB per forward)
    t_off, infos = [], []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record(stream)
        _, info = off.forward(x, y_off, want_timeline=True)
        b.record(stream)
        b.synchronize()
        t_off.append(a.elapsed_time(b))
        infos.append(info)
    t_o = float(np.mean(t_off))
    counts = infos[-1]["counts"]
    # the same layer streaming exph packs (lossless; bit-identical output)
    y_offh = torch.empty_like(x)
    offh.forward(x, y_offh)
    t_offh = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record(stream)
        offh.forward(x, y_offh)
        b.record(stream)
        b.synchronize()
        t_offh.append(a.elapsed_time(b))
    t_oh = float(np.mean(t_offh))
    packed = offh.packed_bytes()
    y_offs = torch.empty_like(x)
    off_skip.forward(x, y_offs)
    t_offs = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record(stream)
        off_skip.forward(x, y_offs)
        b.record(stream)
        b.synchronize()
        t_offs.append(a.elapsed_time(b))
    t_os = float(np.mean(t_offs))
    wbytes = 2 * d * f * 2
    g = im.make_geometry(d, f, E, 2)
    cv = im.compute_costs(counts.astype(np.uint64), g, hw)
    _, sim_rep, _ = im.simulate_model([cv], K)
    # resident: one fused-FFN launch over all 64 experts (tensor-bound)
    t_res = []
    for _ in range(reps):
        a, b = ev(), ev()
        a.record(stream)
        res.forward(x, y_res, want_info=False)
        b.record(stream)
        b.synchronize()
        t_res.append(a.elapsed_time(b))
    _, rinfo = res.forward(x, y_res, want_timeline=True)
    torch.cuda.synchronize()
    ffn_s = rinfo["events"][0][4] - rinfo["events"][0][3]
    flops = 4.0 * N * k * d * f
    hbm_bytes = int((counts > 0).sum()) * wbytes + N * k * (2 * d + 2 * f) * 2
    t_bound = max(flops / (float(peaks["bf16_tflops"]) * 1e12),
                  hbm_bytes / (float(peaks["hbm_gbs"]) * 1e9))
    same = bool(torch.equal(y_off.view(torch.int16), y_res.view(torch.int16)))

    # dispatch / combine kernels at C5 size, each launch after an L2 flush
    flush = _l2_flush(torch, dev)
    idx, w, _ = dv.gate_softmax_topk(x, torch.from_numpy(gw).to(dev), k,
                                     bias=torch.from_numpy(bias).to(dev))
    offs, perm, inv = dv.dispatch(idx, E)
    xp = dv.gather_rows(x, perm, k)
    torch.cuda.synchronize()

    def timed(fn, n=5, back_to_back=8):
        # after an L2 flush, `back_to_back` launches between two events (the
        # per-launch event / launch overhead amortised; every working set here
        # exceeds the 126 MB L2), median over n repetitions
        ts = []
        for _ in range(n):
            flush()
            a, b = ev(), ev()
            a.record(stream)
            for _ in range(back_to_back):
                fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3 / back_to_back)
        return float(np.median(ts))

    wg_dev, b_dev = torch.from_numpy(gw).to(dev), torch.from_numpy(bias).to(dev)
    gws = dv.GateWorkspace(wg_dev, N, k)  # as a layer holds it: W_g split once
    t_gate = timed(lambda: dv.gate_softmax_topk(x, wg_dev, k, bias=b_dev, workspace=gws))
    gstats = dv.gate_softmax_topk(x, wg_dev, k, bias=b_dev, debug=True)[4]
    t_disp = timed(lambda: dv.dispatch(idx, E))
    t_gath = timed(lambda: dv.gather_rows_by_token(x, inv, k))  # the layer's k > 1 path
    t_comb = timed(lambda: dv.combine(xp, inv, w, N, k))
    hbm = float(peaks["hbm_gbs"])
    gath_b = N * d * 2 + N * k * d * 2 + N * k * 4       # x once, x_perm, inv
    comb_b = N * k * d * 2 + N * d * 2 + N * k * 8       # y_perm, y, inv + weights
    gate_b = N * d * 2 + E * d * 4 + N * k * 8            # x, W_g, idx + weights
    mv = {"config": "C5 sizes: 16384 tokens x 4096, top-2, E=64, bf16; per launch = median "
                    "over 5 repetitions of (256 MB L2 flush, 8 launches back to back between "
                    "CUDA events on the launching stream) / 8",
          "ncu": "profiles/r02_dm_ncu_summary.txt (cold-cache, serialised launches)",
          "gate_softmax_topk": {"us": t_gate * 1e6, "gbs": gate_b / t_gate / 1e9,
                                "frac": gate_b / t_gate / 1e9 / hbm,
                                "bytes": gate_b,
                                "path": "tcgen05 logits (W_g = hi + mid + lo bf16) + certified "
                                        "top-k, exact fmaf chains for the uncertified tokens",
                                "certified_tokens": gstats["certified"] if gstats else None,
                                "fallback_tokens": gstats["fallback"] if gstats else None,
                                "exact_chains": gstats["candidates"] if gstats else None},
          "dispatch_counting_sort": {"us": t_disp * 1e6, "assignments": N * k},
          "gather_rows": {"us": t_gath * 1e6, "gbs": gath_b / t_gath / 1e9,
                          "frac": gath_b / t_gath / 1e9 / hbm, "bytes": gath_b,
                          "kernel": "gather_rows_by_token (warp per token: row read once, "
                                    "written to its k positions)",
                          "bytes_formula": "x read once + x_perm written + inv"},
          "combine": {"us": t_comb * 1e6, "gbs": comb_b / t_comb / 1e9,
                      "frac": comb_b / t_comb / 1e9 / hbm, "bytes": comb_b,
                      "bytes_formula": "y_perm read + y written + inv/weights"},
          "peak_gbs": hbm, "peak_src": peaks["_src"]}
    top = np.sort(counts)[::-1]
    out = {
        "workload": c["workload"], "tokens": N, "experts": E, "top_k": k, "K": K,
        "gate": f"softmax top-2, logit bias -c ln(e+1), c = {c_bias:.4f} calibrated to the "
                "Zipf(1) pin",
        "inputs": "SURVEY 8(d) generators at scenario seed S5 = SEED + 500",
        "zipf_pin_top4": [int(v) for v in zipf[:4]],
        "realised_counts": {"max": int(top[0]), "top4": [int(v) for v in top[:4]],
                            "max_vs_zipf_pin": float(top[0] / zipf[0]),
                            "min": int(top[-1]), "mean": float(counts.mean()),
                            "max_over_mean": float(top[0] / counts.mean())},
        "offloaded": {"tokens_per_s": N / (t_o * 1e-3), "ms_per_layer": t_o,
                      "h2d_gbs": E * wbytes / (t_o * 1e-3) / 1e9,
                      "h2d_frac": E * wbytes / (t_o * 1e-3) / 1e9 / h2d_peak,
                      "exposed_copy_ms": 1e3 * float(np.mean([i["exposed_copy_s"] for i in infos])),
                      "simulated_ms": sim_rep.makespan * 1e3,
                      "measured_over_simulated": t_o / (sim_rep.makespan * 1e3),
                      "order_head": [int(v) for v in infos[-1]["order"][:8]],
                      "reps": reps},
        "resident": {"tokens_per_s": N / (float(np.mean(t_res)) * 1e-3),
                     "ms_per_layer": float(np.mean(t_res)),
                     "ffn_us": ffn_s * 1e6,
                     "ffn_tflops": flops / ffn_s / 1e12,
                     "ffn_tensor_frac": flops / ffn_s / 1e12 / float(peaks["bf16_tflops"]),
                     "layer_over_t_bound": t_bound / (float(np.mean(t_res)) * 1e-3),
                     "t_bound_ms": t_bound * 1e3,
                     "bound": "tensor" if flops / (float(peaks["bf16_tflops"]) * 1e12) >=
                     hbm_bytes / (hbm * 1e9) else "hbm"},
        "offloaded_exph": {"tokens_per_s": N / (t_oh * 1e-3), "ms_per_layer": t_oh,
                           "bits_per_weight": 16.0 * packed / (E * wbytes),
                           "h2d_gbs": packed / (t_oh * 1e-3) / 1e9,
                           "h2d_frac": packed / (t_oh * 1e-3) / 1e9 / h2d_peak,
                           "speedup_vs_raw": t_o / t_oh,
                           "bit_identical_to_raw": bool(torch.equal(
                               y_offh.view(torch.int16), y_off.view(torch.int16)))},
        "offloaded_exph_skip_empty": {
            "tokens_per_s": N / (t_os * 1e-3), "ms_per_layer": t_os,
            "experts_loaded": int((counts > 0).sum()), "experts": E,
            "note": "the reference's skip_empty_experts option (default off): experts with no "
                    "rows are neither scheduled nor loaded",
            "bit_identical_to_raw": bool(torch.equal(y_offs.view(torch.int16),
                                                     y_off.view(torch.int16)))},
        "offloaded_bit_identical_to_resident": same,
        "data_movement": mv,
    }
    res.close()
    off.close()
    offh.close()
    off_skip.close()
    return out


def _smi_state(tag):
    q = ("clocks.sm,clocks.mem,power.draw,power.limit,enforced.power.limit,temperature.gpu,"
         "temperature.memory,clocks_event_reasons.active")
    try:
        out = subprocess.run(["nvidia-smi", "--id=0", f"--query-gpu={q}", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=10).stdout.strip()
    except Exception as exc:  # noqa: BLE001
        out = repr(exc)
    print(f"[{tag}] {out}", file=sys.stderr)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--K", type=int, default=None, help="resident experts per layer")
    ap.add_argument("--host-sets", type=int, default=2,
                    help="distinct host weight sets aliased across layers (bytes moved are "
                         "identical; bounds pinned memory)")
    ap.add_argument("--resident-steps", type=int, default=20)
    ap.add_argument("--cpu-sample", type=int, default=1024,
                    help="tokens per CPU pass (cpu_baseline leg and --impl reference): a real "
                         "pass through all layers on this many of the workload's tokens")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pin-frac", type=float, default=0.5,
                    help="hot-expert pinning line (SURVEY 8(f)-4, not reference-faithful): "
                         "fraction of each layer's experts kept on the device (0 skips it)")
    ap.add_argument("--pack-cache", default=None,
                    help="directory of h2d-codec packs (infmoe_set_pack_cache_dir): packs are "
                         "read from it instead of encoded when their content matches, and "
                         "written to it after encoding (default: encode, no files)")
    ap.add_argument("--h2d-codec", default="exph", choices=["exph", "exp4", "raw"],
                    help="exph (default) / exp4: the headline streams lossless packs (Huffman-"
                         "coded or 4-bit exponents, ~10.7 / 12 bits per weight, decoded on the "
                         "GPU, bit-identical outputs) and the raw bf16 stream (the reference's "
                         "expert_param_bytes) is reported beside it as raw_stream; raw: the raw "
                         "stream only")
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the C5 (E64 top-2 skewed, offloaded) and data-movement lines")
    ap.add_argument("--no-continuous", dest="continuous", action="store_false",
                    help="skip the continuous_load_stream line")
    ap.add_argument("--ep-transport", default="nccl", choices=["nccl", "peer"],
                    help="expert-parallel exchange for N > 1: grouped NCCL send/recv, or rows "
                         "pushed over peer memory (CUDA IPC) with the return fused into the FFN")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.K:
        cfg["K"] = args.K

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2106_10715_b200 as im
    from paper_2106_10715_b200 import device as dv

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa = None
    if world > 1:
        numa = bind_to_gpu_numa_node(local)
        dist.init_process_group("nccl", device_id=dev)
    peaks = measured_peaks()
    d, f, E, k, N_glob, L = cfg["d"], cfg["f"], cfg["E"], cfg["k"], cfg["N"], cfg["L"]
    P = world                      # expert parallelism over all ranks (strong scaling)
    if E % P or N_glob % P:
        raise SystemExit(f"experts ({E}) and tokens ({N_glob}) must divide by {P} ranks")
    El, N = E // P, N_glob // P    # experts and tokens owned by this rank
    bf = torch.bfloat16
    stream = torch.cuda.current_stream()
    comm = None
    if P > 1:  # the layers' own NCCL communicator (id shared through torch.distributed)
        uid = [im.ep_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = im.ep_comm_init(uid[0], P, rank)

    # --- pinned H2D peak on this box (roofline denominator for the host link)
    probe_h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    probe_d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    h2d_peak = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        probe_d.copy_(probe_h, non_blocking=True)
        e1.record()
        e1.synchronize()
        h2d_peak = max(h2d_peak, (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    del probe_h, probe_d
    ep_probe = None
    if world > 1:
        # SURVEY 8(d)'s multi-GPU probes: every rank's pinned H2D peak measured
        # CONCURRENTLY (the copies above ran on all ranks at once), and the NCCL
        # all-to-all at the C4 message size (each rank sends (N/P)*k*(P-1)/P rows
        # of d bf16 in total, split evenly over its peers), median of 10
        peaks_all = [None] * world
        dist.all_gather_object(peaks_all, h2d_peak)
        rows_pp = max(1, (N_glob // world) * k // world)
        sbuf = torch.empty(world * rows_pp * d, dtype=torch.bfloat16, device=dev)
        rbuf = torch.empty_like(sbuf)
        for _ in range(3):
            dist.all_to_all_single(rbuf, sbuf)
        ts = []
        for _ in range(10):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dist.all_to_all_single(rbuf, sbuf)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t_a2a = float(np.median(ts))
        tt = torch.tensor([t_a2a], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_a2a = tt.item()
        sent = (world - 1) * rows_pp * d * 2  # bytes each rank sends to its peers
        ep_probe = {"h2d_peak_gbs_per_rank_concurrent": peaks_all,
                    "alltoall": {"bytes_sent_per_rank": sent, "us": t_a2a * 1e6,
                                 "algbw_gbs_per_rank": sent / t_a2a / 1e9,
                                 "how": "torch.distributed all_to_all_single (NCCL) of the C4 "
                                        "dispatch size, max over ranks of the median of 10"}}
        del sbuf, rbuf

    # --- weights: n_sets distinct sets of this rank's experts in
    # one pinned host pool, plus device copies.  Set s is the layer weights of
    # scenario seed S_s = SEED + s: W_in[e] = GaussianStream(derive_seed(S_s,
    # 1000 + 2e)) x d^-1/2, W_out[e] = GaussianStream(derive_seed(S_s, 1001 + 2e))
    # x f^-1/2 (prng.hpp:49-71), rounded to bf16 (f32 RN, then RNE), generated on
    # the host cores (the same values whatever the rank count)
    n_sets = max(1, min(args.host_sets, L))
    per_e = f * d
    host_pool = torch.empty(n_sets * 2 * El * per_e, dtype=bf, pin_memory=True)
    t_gen = time.perf_counter()
    w_dev, w_host = [], []
    for s in range(n_sets):
        base = 2 * s * El * per_e
        hi = host_pool[base:base + El * per_e].view(El, f, d)
        ho = host_pool[base + El * per_e:base + 2 * El * per_e].view(El, d, f)
        fill_expert_weights(im, SEED + s, rank * El, El, d, f, hi, ho)
        w_dev.append((hi.to(dev), ho.to(dev)))
        w_host.append((hi, ho))
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t_gen

    hw = im.Hardware(float(peaks["bf16_tflops"]) * 1e12, h2d_peak * 1e9, 180 << 30, 8 << 30)
    # x = gaussian_tokens(derive_seed(SEED, 0), N, d) (gating.hpp:108-114) in bf16;
    # rank r owns tokens [r N/P, (r+1) N/P)
    x_bits = im.gaussian_bf16(im.derive_seed(SEED, 0), N_glob * d)[rank * N * d:(rank + 1) * N * d]
    x_host = torch.empty((N, d), dtype=bf, pin_memory=True)
    x_host.view(torch.int16).copy_(torch.from_numpy(x_bits.view(np.int16).reshape(N, d)))
    x_dev = x_host.to(dev)
    y_host = torch.empty((N, d), dtype=bf, pin_memory=True)

    # one pool of K+1 expert slots shared by all offloaded layers: K experts on
    # the GPU for the whole stack, as the reference's resident_capacity models it
    pool = dv.SlotPool(cfg["K"], d, f, device=local)

    def make_layers(offloaded: bool):
        out = []
        for l in range(L):
            s = l % n_sets
            wi, wo = (w_host if offloaded else w_dev)[s]
            out.append(dv.MoELayer(d, f, E, k, wi, wo, gate="lsh",
                                   lsh_seed=lsh_seed(im, l), lsh_bits=cfg["bits"],
                                   offloaded=offloaded, K=cfg["K"], max_tokens=N, device=local,
                                   hw=hw, ep_size=P, ep_rank=rank, ep_comm=comm,
                                   ep_transport=args.ep_transport,
                                   slot_pool=pool if offloaded else None))
        return out

    off_layers = make_layers(True)
    res_layers = make_layers(False)
    # the packed-stream layers (headline) are built here, so the one-time host
    # packing and its 16 GB of pinned packs settle before any timed step
    exp_layers = []
    pack_s = 0.0
    if args.h2d_codec != "raw":
        if args.pack_cache:
            im.set_pack_cache_dir(args.pack_cache)
        t0 = time.perf_counter()
        for l in range(L):
            wi, wo = w_host[l % n_sets]
            exp_layers.append(dv.MoELayer(d, f, E, k, wi, wo, gate="lsh",
                                          lsh_seed=lsh_seed(im, l),
                                          lsh_bits=cfg["bits"], offloaded=True, K=cfg["K"],
                                          max_tokens=N, device=local, hw=hw, ep_size=P,
                                          ep_rank=rank, ep_comm=comm,
                                          ep_transport=args.ep_transport, slot_pool=pool,
                                          h2d_codec=args.h2d_codec))
        pack_s = time.perf_counter() - t0

    bufs = [torch.empty((N, d), dtype=bf, device=dev) for _ in range(2)]

    def stack(layers, x, timeline=False, info=True, origin=None):
        infos = []
        cur = x
        for i, layer in enumerate(layers):
            y = bufs[i % 2]
            _, inf = layer.forward(cur, y, want_timeline=timeline, want_info=info or timeline,
                                   time_origin=origin)
            infos.append(inf)
            cur = y
        return cur, infos

    def link_idle_ms(infos, ms_per_step: float) -> float:
        """Host-link idle time per layer in the TIMED steps: the step time minus the
        load lane's busy time (load durations from the untimed timeline step, which
        run at the same rate), per layer.  (The timeline step itself idles longer at
        each layer boundary: collecting a layer's events makes the host wait for the
        layer's end before it issues the next layer.)"""
        busy = sum(e[4] - e[3] for i in infos for e in i["events"] if e[0] == 0)
        return (ms_per_step - 1e3 * busy) / len(infos)

    if os.environ.get("BENCH_VERBOSE"):
        for rep in range(2):
            _, pre = stack(res_layers, x_dev, timeline=True)
        _smi_state("pre")
        for l, i in enumerate(pre[:6]):
            print(f"pre resident layer {l}: ffn {(i['events'][0][4] - i['events'][0][3]) * 1e6:.1f} us",
                  file=sys.stderr)

    # ---------------- offloaded stack: warm-up, then timed steps -------------
    for _ in range(args.warmup):
        stack(off_layers, x_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    inner_ms, outer_ms, all_infos = [], [], []
    with (ClockSampler(local) if not os.environ.get("BENCH_NOSMI") else ClockSampler(-1)) as clocks:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            a, b, c, dd = ev(), ev(), ev(), ev()
            a.record(stream)
            x_dev.copy_(x_host, non_blocking=True)        # H2D of the step's input
            b.record(stream)
            # no timeline in the timed steps: collecting one makes every layer
            # wait for its own end (events read back) before the next is issued
            y, infos = stack(off_layers, x_dev)
            c.record(stream)
            y_host.copy_(y, non_blocking=True)             # D2H of the step's result
            dd.record(stream)
            dd.synchronize()
            inner_ms.append(b.elapsed_time(c))
            outer_ms.append(a.elapsed_time(dd))
    torch.cuda.synchronize()
    # one more step, untimed, with the measured timelines (exposed copy, FFN
    # durations, replay_check, simulator comparison)
    _, diag = stack(off_layers, x_dev, timeline=True)
    all_infos.append(diag)
    t_in = float(np.mean(inner_ms))
    t_out = float(np.mean(outer_ms))
    if world > 1:
        tt = torch.tensor([t_in, t_out], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_in, t_out = tt.tolist()
    y_off = y.clone()

    # per-expert FFN (GEMM pair) durations and exposed copy from the timelines
    ffn_bytes = ffn_secs = 0.0
    exposed = []
    launches = 0
    # dispatch is one single-CTA launch up to 32768 assignments / 128 experts
    dispatch_launches = 1 if N * k <= 32768 and E <= 128 else 3
    wbytes = 2 * d * f * 2
    for infos in all_infos:
        for info in infos:
            rows = info["local_rows"]  # rows this rank computed per local expert
            exposed.append(info["exposed_copy_s"])
            # gate + dispatch + gather + one fused FFN per expert with rows (the top-1
            # combine is fused into it); EP adds the receive-side gather and the combine
            launches += 2 + dispatch_launches + int((rows > 0).sum()) + (2 if P > 1 else 0)
            for (st, _l, e, s0, s1) in info["events"]:
                if st == 1 and rows[e] > 0:
                    ffn_secs += s1 - s0
                    ffn_bytes += wbytes + int(rows[e]) * (2 * d + 2 * f) * 2
    launches //= len(all_infos)
    # the reference simulator's prediction for the realised counts, with the
    # link bandwidth measured on this box (simulate_model, simulator.hpp:241)
    g_loc = im.make_geometry(d, f, El, 2)
    hw_meas = im.Hardware(float(peaks["bf16_tflops"]) * 1e12, h2d_peak * 1e9, 180 << 30, 8 << 30)
    costs = [im.compute_costs(info["local_rows"].astype(np.uint64), g_loc, hw_meas)
             for info in all_infos[-1]]
    _, sim_rep, _ = im.simulate_model(costs, cfg["K"])
    # the measured timelines of the last step against replay_check's rules
    # (verification.hpp:108-206: one lane per stream, causality, <= K experts
    # resident; durations are measured, so they are not compared to alpha/beta)
    audit = {}
    for info, cv in zip(all_infos[-1], costs):
        for kind, n in im.replay_check(info["events"], [cv], cfg["K"],
                                       check_durations=False, tol_s=2e-6).items():
            audit[kind] = audit.get(kind, 0) + n
    if os.environ.get("BENCH_VERBOSE"):
        for l, info in enumerate(all_infos[-1]):
            ld = [(s1 - s0) for (st, _l, _e, s0, s1) in info["events"] if st == 0]
            ce = max(s1 for (st, _l, _e, s0, s1) in info["events"] if st == 1)
            print(f"offloaded layer {l} (set {l % n_sets}): load rate "
                  f"{2 * d * f * 2 * len(ld) / sum(ld) / 1e9:.2f} GB/s, layer {ce * 1e3:.2f} ms",
                  file=sys.stderr)
    h2d_bytes_step = L * El * wbytes          # this rank's host link

    # ---------------- the headline: the same stack streaming lossless packs ----
    # each load copies the expert's pack (exph: ~10.3 bits per weight) and two
    # decoder kernels restore the bf16 slot bit for bit before the FFN
    # (codec.cuh); measured right after the raw stream, before the heavier
    # phases below (resident soak, 64 GB of pinned experts, C5)
    if args.h2d_codec != "raw":
        for _ in range(args.warmup):
            stack(exp_layers, x_dev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ex_ms, ex_out, ex_infos = [], [], []
        with ClockSampler(local) as ex_clocks:
            for _ in range(args.steps):
                torch.cuda.synchronize()
                a, b, c, dd = ev(), ev(), ev(), ev()
                a.record(stream)
                x_dev.copy_(x_host, non_blocking=True)
                b.record(stream)
                y_ex, _ = stack(exp_layers, x_dev)
                c.record(stream)
                y_host.copy_(y_ex, non_blocking=True)
                dd.record(stream)
                dd.synchronize()
                ex_ms.append(b.elapsed_time(c))
                ex_out.append(a.elapsed_time(dd))
        o_ev = torch.cuda.Event(enable_timing=True)
        o_ev.record(stream)
        _, einfos = stack(exp_layers, x_dev, timeline=True, origin=o_ev)  # untimed diagnostics
        ex_infos.append(einfos)
        t_ex, t_ex_out = float(np.mean(ex_ms)), float(np.mean(ex_out))
        if world > 1:
            tt = torch.tensor([t_ex, t_ex_out], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ex, t_ex_out = tt.tolist()
        packed = sum(lay.packed_bytes() for lay in exp_layers[:n_sets])
        raw = n_sets * El * wbytes
        link_bytes = L * El * wbytes * packed / raw  # packed bytes moved per step
        audit_ex = {}
        for info, cv in zip(ex_infos[-1], costs):
            for kind, nv in im.replay_check(info["events"], [cv], cfg["K"],
                                            check_durations=False, tol_s=2e-6).items():
                audit_ex[kind] = audit_ex.get(kind, 0) + nv
        # the reference simulator with the link's effective weight bandwidth
        # (bytes per expert / packed bytes per expert x measured pinned peak)
        hw_eff = im.Hardware(float(peaks["bf16_tflops"]) * 1e12, h2d_peak * 1e9 * raw / packed,
                             180 << 30, 8 << 30)
        costs_eff = [im.compute_costs(i["local_rows"].astype(np.uint64), g_loc, hw_eff)
                     for i in ex_infos[-1]]
        _, sim_eff, _ = im.simulate_model(costs_eff, cfg["K"])
    h2d_gbs = h2d_bytes_step / (t_in * 1e-3) / 1e9

    # ---------------- resident stack (all experts in HBM) --------------------
    # no host round trip on this path (one GPU, or EP over the PEER transport),
    # so the 24-layer stack is captured once as a CUDA graph and replayed; the
    # NCCL transport plans the exchange on the host and runs eagerly.
    graph = None
    for _ in range(3):
        stack(res_layers, x_dev, info=False)
    torch.cuda.synchronize()
    if os.environ.get("BENCH_VERBOSE"):
        _, mid = stack(res_layers, x_dev, timeline=True)
        _smi_state("mid")
        for l, i in enumerate(mid[:4]):
            print(f"mid resident layer {l}: ffn {(i['events'][0][4] - i['events'][0][3]) * 1e6:.1f} us",
                  file=sys.stderr)
    if P == 1 or args.ep_transport == "peer":  # no host round trip: capturable
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            y_graph, _ = stack(res_layers, x_dev, info=False)
        graph.replay()
        torch.cuda.synchronize()
    a, b = ev(), ev()
    with ClockSampler(local) as res_clocks:
        a.record(stream)
        for _ in range(args.resident_steps):
            if graph is not None:
                graph.replay()
                y_res = y_graph
            else:
                y_res, _ = stack(res_layers, x_dev, info=False)
        b.record(stream)
        b.synchronize()
    if os.environ.get("BENCH_VERBOSE"):
        print("resident clocks", res_clocks.summary(), [r[1:4] for r in res_clocks.rows],
              file=sys.stderr)
    t_res = a.elapsed_time(b) / args.resident_steps
    if world > 1:
        tt = torch.tensor([t_res], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_res = tt.item()
    # one timeline pass for the grouped-GEMM share
    _, rinfos = stack(res_layers, x_dev, timeline=True)
    rg_secs = sum(i["events"][0][4] - i["events"][0][3] for i in rinfos)
    if os.environ.get("BENCH_VERBOSE"):
        for l, i in enumerate(rinfos):
            print(f"resident layer {l}: ffn {(i['events'][0][4] - i['events'][0][3]) * 1e6:.1f} us "
                  f"max_rows {int(i['local_rows'].max())}", file=sys.stderr)
    rg_bytes = 0
    for i in rinfos:
        rows = i["local_rows"]
        rg_bytes += int((rows > 0).sum()) * wbytes + int(rows.sum()) * (2 * d + 2 * f) * 2
    parity_equal = bool(torch.equal(y_res.view(torch.int16), y_off.view(torch.int16)))

    # ---------------- sustained FFN: the fused FFN alone, back to back -------
    # one launch per layer (each layer's weight set) on layer 0's routing, the
    # whole sequence as one CUDA graph: the kernel timed inside a long run
    # (power-capped), next to the per-launch timing of the timeline pass
    sustained = None
    if P == 1:
        proj0 = torch.from_numpy(np.ascontiguousarray(
            im.gating_projection(lsh_seed(im, 0), cfg["bits"], d))).to(dev)
        _, idx0, w0, cnt0 = dv.gate_lsh(x_dev, proj0, E)
        off0, perm0, _ = dv.dispatch(idx0, E)
        xp0 = dv.gather_rows(x_dev, perm0, 1)
        torch.cuda.synchronize()
        for _ in range(2):
            for l in range(L):
                dv.expert_ffn_fused(xp0, off0, *w_dev[l % n_sets], perm=perm0,
                                    topk_w=w0.reshape(-1), n_tokens=N)
        torch.cuda.synchronize()
        gf = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gf):
            for l in range(L):
                dv.expert_ffn_fused(xp0, off0, *w_dev[l % n_sets], perm=perm0,
                                    topk_w=w0.reshape(-1), n_tokens=N)
        gf.replay()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        with ClockSampler(local) as ffn_clocks:
            a.record(stream)
            for _ in range(3):
                gf.replay()
            b.record(stream)
            b.synchronize()
        t_launch = a.elapsed_time(b) / (3 * L) * 1e-3
        c0 = cnt0.cpu().numpy()
        sb = int((c0 > 0).sum()) * wbytes + int(c0.sum()) * (2 * d + 2 * f) * 2
        sustained = {"achieved": sb / t_launch / 1e9, "frac": sb / t_launch / 1e9 / float(peaks["hbm_gbs"]),
                     "us_per_launch": t_launch * 1e6, "launches_timed": 3 * L,
                     "how": f"{L} fused-FFN launches back to back in one CUDA graph (layer 0's "
                            "routing, each layer's weights), replayed 3x, CUDA events",
                     "clocks": ffn_clocks.summary()}
        del gf

    # ---------------- CPU baseline (rank 0, N=1 only) ------------------------
    # (1) timed: the CPU path (oracle/cpu_stack.py, the same code as --impl
    #     reference) over a token sample through all L layers, on the weights the
    #     GPU streams; (2) parity: the GPU's layer 0 on ALL N tokens against the
    #     fp64 CPU oracle (the checker)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
        cs = _cpu_stack_module()
        n_tok = min(args.cpu_sample, N)
        bits_of = lambda t: t.view(torch.int16).numpy().view(np.uint16)
        w_sets = [(bits_of(hi), bits_of(ho)) for hi, ho in w_host]
        xb = bits_of(x_host).reshape(N, d)
        cpu_stack = cs.CpuStack(d, f, E, cfg["bits"], cfg["K"],
                                [lsh_seed(im, l) for l in range(L)], w_sets,
                                float(peaks["bf16_tflops"]) * 1e12, h2d_peak * 1e9)
        t0 = time.perf_counter()
        y_cpu = cpu_stack.forward(np.ascontiguousarray(xb[:n_tok]), L)
        t_cpu = time.perf_counter() - t0
        yg_stack = bits_of(y_off.cpu())[:n_tok]
        f32 = lambda b: (b.astype(np.uint32) << 16).view(np.float32)
        e_stack = np.abs(f32(yg_stack) - f32(y_cpu))
        row_ok = np.all(e_stack <= 3e-2 * np.abs(f32(y_cpu)).max() + 2e-2 * np.abs(f32(y_cpu)),
                        axis=1)
        # parity of the GPU's layer 0 on all N tokens (fp64 oracle)
        y0, info0 = res_layers[0].forward(x_dev, torch.empty_like(x_dev))
        _, idx_s, _, _ = dv.gate_lsh(x_dev, proj0, E)
        _, perm_s, _ = dv.dispatch(idx_s, E)
        torch.cuda.synchronize()
        par = layer0_parity(cfg, xb, w_sets[0][0].reshape(E, -1), w_sets[0][1].reshape(E, -1),
                            np.ascontiguousarray(im.gating_projection(lsh_seed(im, 0),
                                                                      cfg["bits"], d)),
                            y0.float().cpu().numpy(), info0["counts"], perm_s.cpu().numpy())
        cpu = {"value": n_tok / t_cpu, "unit": "tokens/s", "cores": cs.cpu_threads(),
               "kind": "port", "cpu": cs.cpu_model(),
               "sample": f"the first {n_tok} of the {N} tokens through all {L} layers "
                         f"(one real pass, {t_cpu:.2f} s)",
               "path": "oracle/cpu_stack.py (same as --impl reference): reference lsh_codes "
                       "and auto_order (oracle/_ref), port dispatch / bf16 FFN with fp32 "
                       f"accumulation ({cpu_stack.isa}) / combine",
               "stack_output_vs_gpu": {
                   "rows": int(n_tok),
                   "rows_within_tol_frac": float(row_ok.mean()),
                   "median_abs_err": float(np.median(e_stack)),
                   "note": "after 24 layers a token whose LSH sign flips between the two "
                           "accumulation orders takes another expert, so rows are compared "
                           "whole; layer-0 parity below is the bit-exact / tolerance check"},
               # the GPU layer 0 on all N tokens against the fp64 oracle
               "parity": par}

    hbm_peak = float(peaks["hbm_gbs"])
    traffic = None  # DRAM bytes per launch of the same kernel from the committed ncu capture
    tp = ROOT / "profiles" / "r02_ffn_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("traffic_bytes_per_launch")
    ffn_gbs = ffn_bytes / ffn_secs / 1e9 if ffn_secs else 0.0
    rg_gbs = rg_bytes / rg_secs / 1e9 if rg_secs else 0.0
    value = N_glob / (t_in * 1e-3)
    line = {
        "metric": "moe_stack_tokens_per_s", "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_in,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic: SURVEY 8(d) generators (gaussian_tokens x, GaussianStream expert "
                "weights x d^-1/2 / f^-1/2; the reference's prng.hpp stream, bit-exact), "
                "random-init weights",
        "config": bench_config(cfg, args, P, n_sets),
        "input_generation_s": gen_s,
        "e2e": {"value": N_glob / (t_out * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": N * d * 2, "d2h_bytes_per_step": N * d * 2},
        "h2d": {"achieved_gbs": h2d_gbs, "peak_gbs": h2d_peak, "frac": h2d_gbs / h2d_peak,
                "bytes_per_step": h2d_bytes_step, "peak_src": "measured pinned 1 GiB copy",
                "per": "rank (each rank streams its own experts over its own host link)",
                "exposed_copy_ms_per_layer": 1e3 * float(np.mean(exposed)),
                "simulated_ms_per_step": sim_rep.makespan * 1e3,
                "measured_over_simulated": t_in / (sim_rep.makespan * 1e3),
                "replay_check_violations": audit},
        # dominant kernel of the path: the expert FFN (both tcgen05 projections in
        # one persistent launch), timed with CUDA events on its stream over the
        # resident 24-layer pass; bytes = weights of routed experts + activations
        "roofline": {"kernel": "fused expert FFN (tcgen05 GEMM1+GeLU -> GEMM2 [+top-1 combine]), "
                               "all local experts in one launch",
                     "bound": "hbm", "achieved": rg_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": rg_gbs / hbm_peak, "traffic": traffic,
                     "traffic_src": "profiles/r02_ffn_traffic.json (ncu dram__bytes_read+write)",
                     "bytes_per_launch": rg_bytes / max(1, len(rinfos)),
                     "launches_timed": len(rinfos), "peak_src": peaks["_src"],
                     "timing": "per-launch CUDA events in a 24-layer resident pass that reads "
                               "routing counts back after each layer (brief idle gaps)",
                     "sustained": sustained},
        "offloaded_ffn": {"kernel": "same kernel, one expert per launch behind each H2D copy "
                                    "(off the critical path: the host link binds)",
                          "achieved_gbs": ffn_gbs, "frac": ffn_gbs / hbm_peak},
        "resident": {"tokens_per_s": N_glob / (t_res * 1e-3), "ms_per_step": t_res,
                     "cuda_graph": graph is not None,
                     "ms_per_layer": t_res / L,
                     "grouped_ffn_share": rg_secs * 1e3 / t_res if t_res else None,
                     "bit_identical_to_offloaded": parity_equal,
                     "clocks": res_clocks.summary()},
        "gpu_launches": launches,
        "ep_probe": ep_probe,
        "cpu_affinity": numa,
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    # ---------------- hot-expert pinning (reported apart) -------
    # the same offloaded stack with the hottest pin_frac of each layer's experts
    # (by the last timed step's counts) kept on the device across steps: those
    # need no H2D, the rest stream in the InfMoE order over their own costs
    n_pin = int(round(args.pin_frac * El))
    if n_pin > 0:
        for lay in off_layers:  # the layer's cache policy: EMA of routed rows over forwards
            lay.pin_hottest(n_pin)
        stack(off_layers, x_dev)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        pin_ms, pin_infos = [], []
        for _ in range(args.steps):
            a, b = ev(), ev()
            a.record(stream)
            y_pin, pinfos = stack(off_layers, x_dev, timeline=True)
            b.record(stream)
            b.synchronize()
            pin_ms.append(a.elapsed_time(b))
            pin_infos.append(pinfos)
        t_pin = float(np.mean(pin_ms))
        if world > 1:
            tt = torch.tensor([t_pin], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_pin = tt.item()
        streamed = sum(len([e for e in i["events"] if e[0] == 0]) for i in pin_infos[-1])
        line["pinned"] = {
            "note": "NOT reference-faithful (moesim evicts every expert at compute end, "
                    "SPEC.md:325): SURVEY 8(f)-4 hot-expert pinning, reported apart",
            "tokens_per_s": N_glob / (t_pin * 1e-3), "ms_per_step": t_pin,
            "pinned_per_layer": n_pin, "experts_per_layer": El,
            "device_bytes_pinned": L * n_pin * wbytes,
            "h2d_bytes_per_step": streamed * wbytes,
            "h2d_gbs": streamed * wbytes / (t_pin * 1e-3) / 1e9,
            "speedup_vs_offloaded": t_in / t_pin,
            "bit_identical_to_offloaded": bool(torch.equal(y_pin.view(torch.int16),
                                                           y_off.view(torch.int16))),
            "policy": "infmoe_layer_pin_hottest: the experts of each layer with the highest "
                      "EMA (decay 0.5) of routed rows over the warm-up and timed steps"}
        for lay in off_layers:
            lay.pin_experts([])
    if exp_layers:
        raw_stream = {
            "note": "the reference's model: every expert streamed as raw bf16 "
                    "(expert_param_bytes per load), same layers, same order",
            "value": line["value"], "ms_per_step": line["ms_per_step"], "e2e": line["e2e"],
            "h2d": line["h2d"], "gpu_launches": line["gpu_launches"], "clocks": line["clocks"]}
        line["value"] = N_glob / (t_ex * 1e-3)
        line["ms_per_step"] = t_ex
        line["e2e"] = {"value": N_glob / (t_ex_out * 1e-3), "unit": "tokens/s",
                       "h2d_bytes_per_step": N * d * 2, "d2h_bytes_per_step": N * d * 2}
        codec_desc = {
            "exp4": "exp4 (lossless: the same bf16 weights packed once on the host -- a "
                    "sign/mantissa byte and a 4-bit exponent code per value against a "
                    "per-32768-value base, exceptions listed -- decoded on the GPU before "
                    "each expert's FFN; outputs bit-identical to the raw stream)",
            "exph": "exph (lossless: the same bf16 weights packed once on the host -- per "
                    "value a canonical Huffman code (<= 12 bits, one table per matrix) of "
                    "(exponent distance to a per-32768-value or matrix-wide base, top two "
                    "mantissa bits) plus the raw sign and low five mantissa bits, 256-value "
                    "chunks with recorded start bits, 256-byte aligned pack parts -- decoded "
                    "on the GPU before each expert's FFN, the last expert's W_in while its "
                    "W_out is on the link; outputs bit-identical to the raw stream)"}
        line["h2d"] = {
            "codec": codec_desc[args.h2d_codec],
            "achieved_gbs": link_bytes / (t_ex * 1e-3) / 1e9, "peak_gbs": h2d_peak,
            "frac": link_bytes / (t_ex * 1e-3) / 1e9 / h2d_peak,
            "bytes_per_step": link_bytes, "raw_bytes_per_step": h2d_bytes_step,
            "bytes_per_weight": 2.0 * packed / raw,
            "effective_weight_gbs": h2d_bytes_step / (t_ex * 1e-3) / 1e9,
            "peak_src": "measured pinned 1 GiB copy",
            "per": "rank (each rank streams its own experts over its own host link)",
            "exposed_copy_ms_per_layer": 1e3 * float(np.mean(
                [i["exposed_copy_s"] for st in ex_infos for i in st])),
            "simulated_ms_per_step": sim_eff.makespan * 1e3,
            "simulated_with": "simulate_model, beta = expert_param_bytes / (pinned peak x "
                              "raw/packed bytes)",
            "measured_over_simulated": t_ex / (sim_eff.makespan * 1e3),
            "replay_check_violations": audit_ex,
            "link_idle_ms_per_layer": link_idle_ms(ex_infos[-1], t_ex),
            # the copies' own rate in the timeline step (pack bytes / summed load
            # durations): separates a slower link from idle gaps between copies
            "load_lane_gbs": link_bytes / max(1e-12, sum(
                e[4] - e[3] for i in ex_infos[-1] for e in i["events"] if e[0] == 0)) / 1e9,
            "bit_identical_to_raw_stream": bool(torch.equal(y_ex.view(torch.int16),
                                                            y_off.view(torch.int16))),
            "pack_seconds_host_once": pack_s,
            "pack_source": exp_layers[0].pack_source()}
        line["clocks"] = ex_clocks.summary()
        line["gpu_launches"] = line["gpu_launches"] + 2 * L * El  # two decodes per expert
        line["speedup_vs_raw_stream"] = t_in / t_ex
        line["raw_stream"] = raw_stream
        if n_pin > 0 and "pinned" in line:  # both: pinned hot experts + packed stream
            for lay in exp_layers:
                lay.pin_hottest(n_pin)
            stack(exp_layers, x_dev)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            pe = []
            for _ in range(args.steps):
                a, b = ev(), ev()
                a.record(stream)
                y_pe, _ = stack(exp_layers, x_dev)
                b.record(stream)
                b.synchronize()
                pe.append(a.elapsed_time(b))
            t_pe = float(np.mean(pe))
            if world > 1:
                tt = torch.tensor([t_pe], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_pe = tt.item()
            line["pinned"]["with_packed_stream"] = {
                "tokens_per_s": N_glob / (t_pe * 1e-3), "ms_per_step": t_pe,
                "codec": args.h2d_codec,
                "bit_identical_to_offloaded": bool(torch.equal(y_pe.view(torch.int16),
                                                               y_off.view(torch.int16)))}
        # ------------- continuous_load_stream (the reference's option, default off) --
        # the same packed stack with the load lane flowing into the next layer:
        # each layer's predicted first expert is streamed while the previous
        # layer's tail (last decode + FFN, next gate / dispatch / plan) runs
        if args.continuous and P == 1:  # (one GPU: the speculative lane is measured here)
            cpool = dv.SlotPool(cfg["K"], d, f, device=local, sets=2)
            cont = []
            for l in range(L):
                wi, wo = w_host[l % n_sets]
                cont.append(dv.MoELayer(d, f, E, k, wi, wo, gate="lsh", lsh_seed=lsh_seed(im, l),
                                        lsh_bits=cfg["bits"], offloaded=True, K=cfg["K"],
                                        max_tokens=N, device=local, hw=hw, ep_size=P,
                                        ep_rank=rank, ep_comm=comm,
                                        ep_transport=args.ep_transport, slot_pool=cpool,
                                        h2d_codec=args.h2d_codec, continuous_load_stream=True,
                                        prefetch_depth=1))
            for l in range(L):
                cont[l].set_next(cont[(l + 1) % L])  # the next batch's layer 0 follows layer L-1
            for _ in range(args.warmup):
                stack(cont, x_dev)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            cms = []
            for _ in range(max(3, min(args.steps, 5))):
                a, b = ev(), ev()
                a.record(stream)
                y_c, _ = stack(cont, x_dev)
                b.record(stream)
                b.synchronize()
                cms.append(a.elapsed_time(b))
            t_c = float(np.mean(cms))
            if world > 1:
                tt = torch.tensor([t_c], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_c = tt.item()
            o_ev = torch.cuda.Event(enable_timing=True)
            o_ev.record(stream)
            _, cinfos = stack(cont, x_dev, timeline=True, origin=o_ev)
            audit_c = {}
            for info, cv in zip(cinfos, costs_eff):
                for kind, nv in im.replay_check(info["events"], [cv], cfg["K"],
                                                check_durations=False, tol_s=2e-6).items():
                    audit_c[kind] = audit_c.get(kind, 0) + nv
            _, sim_c, _ = im.simulate_model(costs_eff, cfg["K"], continuous_load_stream=True)
            line["continuous_load_stream"] = {
                "note": "the reference's continuous_load_stream option (simulator.hpp:131-133, "
                        "default off = the headline's drain mode), realised speculatively: "
                        "each layer streams the next layer's predicted first expert (EMA of its "
                        "routed rows, InfMoE order) into that layer's own slot set",
                "tokens_per_s": N_glob / (t_c * 1e-3), "ms_per_step": t_c,
                "speedup_vs_drain": t_ex / t_c,
                "prefetch_hits": sum(i["prefetched"] for i in cinfos), "layers": L,
                "saved_ms_per_layer": (t_ex - t_c) / L,
                "link_idle_ms_per_layer_drain": link_idle_ms(ex_infos[-1], t_ex),
                "simulated_ms_per_step": sim_c.makespan * 1e3,
                "measured_over_simulated": t_c / (sim_c.makespan * 1e3),
                "replay_check_violations": audit_c,
                "bit_identical_to_drain": bool(torch.equal(y_c.view(torch.int16),
                                                           y_ex.view(torch.int16)))}
            for lay in cont:
                lay.close()
            cpool.close()
        for lay in exp_layers:
            lay.close()
        del exp_layers
    for lay in off_layers + res_layers:
        lay.close()
    pool.close()
    if world == 1 and not args.no_c5:
        # BASELINE.json configs[4] on this GPU, after the headline's buffers are freed
        del off_layers, res_layers, w_dev, w_host, host_pool, bufs, hi, ho
        graph = y_graph = y_res = y_off = y = None  # noqa: F841
        torch.cuda.empty_cache()
        line["c5"] = measure_c5(torch, im, dv, dev, local, stream, peaks, h2d_peak)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        im.ep_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
