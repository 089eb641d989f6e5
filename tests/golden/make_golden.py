"""Generate tests/golden/*.json from the REFERENCE itself.

Runs the unmodified moesim headers (compiled in place by oracle/Makefile into
oracle/_ref/libmoesim_ref.so) on fixed inputs and freezes the outputs, so the
oracle and the product can be checked on machines without /root/reference.
Usage (container with /root/reference):  python tests/golden/make_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import REF, EventRec, ReportRec, f64a, i32a, ptr  # noqa: E402

assert REF is not None, "oracle/_ref/libmoesim_ref.so is required (build it with make -C oracle)"


def sched(alphas, beta, K, policy, max_T=12):
    a = f64a(alphas)
    o = np.zeros(len(a), np.int32)
    f, d, m = C.c_int(), C.c_int(), C.c_int()
    rc = REF.ref_schedule(ptr(a), len(a), beta, K, {"auto": 0, "greedy": 1, "exact": 2,
                                                     "naive": 3}[policy], max_T, ptr(o),
                          C.byref(f), C.byref(d), C.byref(m))
    return {"rc": rc, "order": o.tolist(), "feasible": bool(f.value), "diagnosis": d.value,
            "method": m.value}


def check(order, alphas, beta, K):
    a = f64a(alphas)
    o = i32a(order)
    s = np.zeros(len(a), np.float64)
    f, vp, vs = C.c_int(), C.c_int(), C.c_int()
    rc = REF.ref_check_constraints(ptr(o), ptr(a), len(a), beta, K, ptr(s), C.byref(f),
                                   C.byref(vp), C.byref(vs))
    return {"rc": rc, "feasible": bool(f.value), "slack": s.tolist(), "viol_pos": vp.value,
            "viol_side": vs.value}


def sim_model(layers, K, mode, policy, continuous, max_T=12):
    Ts = i32a([len(a) for a, _ in layers])
    al = f64a(np.concatenate([f64a(a) for a, _ in layers]))
    be = f64a([b for _, b in layers])
    tot = int(Ts.sum())
    orders = np.zeros(tot, np.int32)
    ev = (EventRec * (2 * tot))()
    rep = ReportRec()
    rc = REF.ref_simulate_model(len(Ts), ptr(Ts), ptr(al), ptr(be), K, mode,
                                {"greedy": 0, "naive": 1, "exact": 2}[policy], int(continuous),
                                max_T, ptr(orders), ev, C.byref(rep))
    return {"rc": rc, "orders": orders.tolist(),
            "events": [[e.stream, e.layer_id, e.expert_id, e.start, e.end] for e in ev],
            "report": [rep.makespan, rep.compute_busy, rep.load_busy, rep.compute_stall,
                       rep.peak_resident, rep.overlap_efficiency]}


def main() -> None:
    g = {}
    # ---- prng (prng.hpp) ----
    g["mt64_first"] = {str(s): int(REF.ref_mt64_first(s)) for s in (0, 1, 5489, 2**63 + 7)}
    g["splitmix64"] = {str(s): int(REF.ref_splitmix64(s)) for s in (0, 1, 42, 2**64 - 1)}
    g["derive_seed"] = [[s, t, int(REF.ref_derive_seed(s, t))]
                        for s, t in ((1, 0), (20261018, 0), (0, 1), (7, 1000), (7, 1001))]
    toks = np.zeros(3 * 7, np.float64)
    REF.ref_gaussian_tokens(0, 3, 7, ptr(toks))
    g["gaussian_tokens_seed0_3x7"] = toks.tolist()
    proj = np.zeros(5 * 768, np.float64)
    assert REF.ref_gating_projection(0, 5, 768, ptr(proj)) == 0
    g["gating_projection_seed0_5x768_sample"] = {str(i): proj[i] for i in (0, 1, 2, 767, 768,
                                                                           3839)}
    # ---- LSH gate (gating.hpp:61-104) on small reference inputs ----
    lsh = []
    for seed, n, dim, bits, E in ((3, 64, 96, 3, 8), (11, 200, 128, 5, 32), (5, 50, 33, 6, 40),
                                  (9, 17, 768, 5, 32)):
        x = np.zeros(n * dim, np.float64)
        REF.ref_gaussian_tokens(seed, n, dim, ptr(x))
        codes = np.zeros(n, np.uint32)
        assert REF.ref_lsh_codes(seed + 100, bits, dim, ptr(x), n, ptr(codes)) == 0
        counts = np.zeros(E, np.uint64)
        assert REF.ref_route_tokens(seed + 100, bits, dim, ptr(x), n, E, ptr(counts)) == 0
        lsh.append({"x_seed": seed, "n": n, "dim": dim, "proj_seed": seed + 100, "bits": bits,
                    "E": E, "codes": codes.tolist(), "counts": counts.tolist()})
    g["lsh"] = lsh
    # ---- synthetic workloads (gating.hpp:116-165) ----
    wl = []
    for kind, total, E, seed, s in ((2, 64, 4, 0, 1.0), (2, 5, 2, 0, 1.0), (0, 1000, 7, 3, 1.0),
                                    (1, 10000, 8, 1, 1.0), (1, 32768, 64, 1, 1.0),
                                    (1, 4096, 32, 9, 1.3)):
        c = np.zeros(E, np.uint64)
        assert REF.ref_synthetic_workload(kind, total, E, seed, s, ptr(c)) == 0
        wl.append({"kind": kind, "total": total, "E": E, "seed": seed, "zipf_s": s,
                   "counts": c.tolist()})
    g["workloads"] = wl
    # ---- cost model (cost_model.hpp) ----
    g["expert_param_bytes"] = [[4096, 10240, 2, int(REF.ref_expert_param_bytes(4096, 10240, 2))],
                               [768, 3072, 4, int(REF.ref_expert_param_bytes(768, 3072, 4))],
                               [1, 1, 1, int(REF.ref_expert_param_bytes(1, 1, 1))]]
    g["expert_flops"] = [[4096, 10240, 1, int(REF.ref_expert_flops(4096, 10240, 1))],
                         [4096, 10240, 4096, int(REF.ref_expert_flops(4096, 10240, 4096))]]
    costs = []
    for counts, peak, bw, (d, f, b) in (([940, 505, 321, 0], 1643.6e12, 55.5e9, (4096, 10240, 2)),
                                        ([3, 2], 1e12, 16e9, (4096, 10240, 2)),
                                        ([10, 0, 7], 3e11, 1e9, (768, 3072, 4))):
        a = np.zeros(len(counts), np.float64)
        beta = C.c_double()
        c = np.asarray(counts, np.uint64)
        assert REF.ref_compute_costs(d, f, b, peak, bw, ptr(c), len(c), ptr(a), C.byref(beta)) == 0
        costs.append({"counts": counts, "peak": peak, "bw": bw, "geom": [d, f, b],
                      "alphas": a.tolist(), "beta": beta.value})
    g["costs"] = costs
    K = C.c_int()
    assert REF.ref_resident_capacity(4096, 10240, 2, 16 << 30, 8 << 30, C.byref(K)) == 0
    g["resident_capacity_spec"] = K.value
    g["resident_capacity_too_small"] = REF.ref_resident_capacity(4096, 10240, 2, 100, 10,
                                                                 C.byref(K))
    # ---- scheduler instances ----
    rng = np.random.default_rng(20261018)
    inst = [([0.5, 2, 1, 0.5], 1.0, 2), ([0, 0, 0], 1.0, 1), ([10, 0, 0, 0, 0], 1.0, 1),
            ([1, 1, 1], 1.0, 3), ([1.5, 1, 1.25, 1], 1.0, 2), ([2, 2], 1.0, 1), ([3.0], 1.0, 1)]
    for _ in range(300):
        T = int(rng.integers(1, 13))
        beta = float(rng.uniform(0.1, 3.0))
        inst.append((rng.uniform(0, 3 * beta, T).tolist(), beta, int(rng.integers(1, 9))))
    for _ in range(60):  # PCIe-regime shaped: T=32/64, tiny alphas, ties
        T = int(rng.choice([32, 64]))
        counts = rng.integers(0, 300, T)
        counts[rng.integers(0, T, 4)] = counts[0]  # force ties
        a = (counts * 167772160.0) / 1643.6e12
        inst.append((a.tolist(), 167772160 * 2 / 55.5e9, int(rng.integers(1, 9))))
    sched_cases = []
    for a, beta, K in inst:
        ok = check(list(range(len(a))), a, beta, K)
        sched_cases.append({"alphas": a, "beta": beta, "K": K,
                            "auto": sched(a, beta, K, "auto"), "greedy": sched(a, beta, K, "greedy"),
                            "exact": sched(a, beta, K, "exact") if len(a) <= 12 else None,
                            "naive": sched(a, beta, K, "naive"), "check_identity": ok,
                            "diagnose": REF.ref_diagnose(ptr(f64a(a)), len(a), beta, K, 12),
                            "digest": "%016x" % REF.ref_instance_digest(ptr(f64a(a)), len(a),
                                                                         beta, K),
                            "lower_bound": REF.ref_lower_bound(ptr(f64a(a)), len(a), beta)})
    g["schedules"] = sched_cases
    # ---- simulator ----
    sims = []
    fig3 = ([0.5, 2, 1, 0.5], 1.0)
    for mode in (0, 1):
        for pol in ("greedy", "naive", "exact"):
            sims.append({"layers": [fig3], "K": 2, "mode": mode, "policy": pol, "continuous": 0,
                         **sim_model([fig3], 2, mode, pol, False)})
    two = ([1.5, 1, 1.25, 1], 1.0)
    for cont in (0, 1):
        sims.append({"layers": [two, two], "K": 2, "mode": 0, "policy": "greedy",
                     "continuous": cont, **sim_model([two, two], 2, 0, "greedy", bool(cont))})
    for _ in range(40):
        L = int(rng.integers(1, 5))
        layers = []
        for _ in range(L):
            T = int(rng.integers(1, 10))
            beta = float(rng.uniform(0.5, 2.0))
            layers.append((rng.uniform(0, 3 * beta, T).tolist(), beta))
        K = int(rng.integers(1, 6))
        mode = int(rng.integers(0, 2))
        cont = int(rng.integers(0, 2))
        pol = str(rng.choice(["greedy", "naive"]))
        sims.append({"layers": layers, "K": K, "mode": mode, "policy": pol, "continuous": cont,
                     **sim_model(layers, K, mode, pol, bool(cont))})
    g["simulations"] = sims
    out = HERE / "moesim_reference.json"
    out.write_text(json.dumps(g, indent=None, separators=(",", ":")))
    print(f"wrote {out} ({out.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
