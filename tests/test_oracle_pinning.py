"""Pin the CPU oracle before trusting it: oracle/oracle.c against the golden
vectors frozen from the reference (tests/golden/moesim_reference.json, made by
tests/golden/make_golden.py from the unmodified moesim headers) and, where
the compiled reference is present, against it live on random instances."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import O, REF, EventRec, ReportRec, f64a, i32a, ptr, schedule

G = json.loads((Path(__file__).parent / "golden" / "moesim_reference.json").read_text())


def test_prng_anchors():
    for s, v in G["mt64_first"].items():
        assert O.or_mt64_first(int(s)) == v
    for s, v in G["splitmix64"].items():
        assert O.or_splitmix64(int(s)) == v
    for s, t, v in G["derive_seed"]:
        assert O.or_derive_seed(s, t) == v
    x = np.zeros(21)
    O.or_gaussian_fill(0, ptr(x), 21)
    assert x.tolist() == G["gaussian_tokens_seed0_3x7"]
    p = np.zeros(5 * 768)
    assert O.or_gating_projection(0, 5, 768, ptr(p)) == 0
    for i, v in G["gating_projection_seed0_5x768_sample"].items():
        assert p[int(i)] == v
    # SURVEY Appendix A anchors
    assert O.or_mt64_first(0) == 2947667278772165694
    assert O.or_derive_seed(1, 0) == 627405149472732430


def test_lsh_codes_and_route_tokens():
    for case in G["lsh"]:
        n, dim = case["n"], case["dim"]
        x = np.zeros(n * dim)
        O.or_gaussian_fill(case["x_seed"], ptr(x), n * dim)
        codes = np.zeros(n, np.uint32)
        assert O.or_lsh_codes(case["proj_seed"], case["bits"], dim, ptr(x), n, ptr(codes)) == 0
        assert codes.tolist() == case["codes"]
        counts = np.zeros(case["E"], np.uint64)
        assert O.or_route_tokens(case["proj_seed"], case["bits"], dim, ptr(x), n, case["E"],
                                 ptr(counts)) == 0
        assert counts.tolist() == case["counts"]


def test_synthetic_workloads():
    for w in G["workloads"]:
        c = np.zeros(w["E"], np.uint64)
        assert O.or_synthetic_workload(w["kind"], w["total"], w["E"], w["seed"], w["zipf_s"],
                                       ptr(c)) == 0
        assert c.tolist() == w["counts"]


def test_cost_model():
    for d, f, b, v in G["expert_param_bytes"]:
        assert O.or_expert_param_bytes(d, f, b) == v
    for d, f, n, v in G["expert_flops"]:
        assert O.or_expert_flops(d, f, n) == v
    for c in G["costs"]:
        a = np.zeros(len(c["counts"]))
        beta = C.c_double()
        cnt = np.asarray(c["counts"], np.uint64)
        d, f, b = c["geom"]
        assert O.or_compute_costs(d, f, b, c["peak"], c["bw"], ptr(cnt), len(cnt), ptr(a),
                                  C.byref(beta)) == 0
        assert a.tolist() == c["alphas"] and beta.value == c["beta"]
    K = C.c_int()
    assert O.or_resident_capacity(4096, 10240, 2, 16 << 30, 8 << 30, C.byref(K)) == 0
    assert K.value == G["resident_capacity_spec"] == 51
    assert O.or_resident_capacity(4096, 10240, 2, 100, 10, C.byref(K)) == 3


def test_schedules_match_reference_golden():
    for s in G["schedules"]:
        a, beta, K = s["alphas"], s["beta"], s["K"]
        rc, order, feas, diag, meth = schedule("or", a, beta, K, "greedy")
        assert (order, feas, diag) == (s["greedy"]["order"], s["greedy"]["feasible"],
                                       s["greedy"]["diagnosis"])
        rc, order, feas, diag, meth = schedule("or", a, beta, K, "auto")
        assert (order, feas, diag, meth) == (s["auto"]["order"], s["auto"]["feasible"],
                                             s["auto"]["diagnosis"], s["auto"]["method"])
        if s["exact"] is not None:
            rc, order, feas, diag, meth = schedule("or", a, beta, K, "exact")
            assert (order, feas, diag) == (s["exact"]["order"], s["exact"]["feasible"],
                                           s["exact"]["diagnosis"])
        assert O.or_diagnose(ptr(f64a(a)), len(a), beta, K, 12) == s["diagnose"]
        assert "%016x" % O.or_instance_digest(ptr(f64a(a)), len(a), beta, K) == s["digest"]
        assert O.or_lower_bound(ptr(f64a(a)), len(a), beta) == s["lower_bound"]
        sl = np.zeros(len(a))
        f, vp, vs = C.c_int(), C.c_int(), C.c_int()
        O.or_check_constraints(ptr(i32a(range(len(a)))), ptr(f64a(a)), len(a), beta, K, ptr(sl),
                               C.byref(f), C.byref(vp), C.byref(vs))
        ci = s["check_identity"]
        assert (bool(f.value), sl.tolist(), vp.value, vs.value) == (
            ci["feasible"], ci["slack"], ci["viol_pos"], ci["viol_side"])


def _oracle_sim(layers, K, mode, policy, cont):
    orders = []
    for a, beta in layers:
        if policy == "naive":
            orders += list(range(len(a)))
        else:
            orders += schedule("or", a, beta, K, "auto" if policy == "greedy" else "exact")[1]
    Ts = i32a([len(a) for a, _ in layers])
    al = f64a(np.concatenate([f64a(a) for a, _ in layers]))
    be = f64a([b for _, b in layers])
    tot = int(Ts.sum())
    ev = (EventRec * (2 * tot))()
    rep = ReportRec()
    assert O.or_run_layers(len(Ts), ptr(Ts), ptr(i32a(orders)), ptr(al), ptr(be), K, mode, cont,
                           ev, C.byref(rep), None, None) == 0
    return orders, [[e.stream, e.layer_id, e.expert_id, e.start, e.end] for e in ev], \
        [rep.makespan, rep.compute_busy, rep.load_busy, rep.compute_stall, rep.peak_resident,
         rep.overlap_efficiency]


def test_simulations_match_reference_golden():
    for s in G["simulations"]:
        layers = [(a, b) for a, b in s["layers"]]
        orders, events, report = _oracle_sim(layers, s["K"], s["mode"], s["policy"],
                                             s["continuous"])
        assert orders == s["orders"]
        assert events == s["events"]
        assert report == s["report"]


@pytest.mark.skipif(REF is None, reason="compiled reference not present")
def test_oracle_vs_reference_random_live():
    rng = np.random.default_rng(7)
    for _ in range(500):
        T = int(rng.integers(1, 40))
        beta = float(rng.uniform(0.01, 2.0))
        a = rng.uniform(0, 3 * beta, T)
        if rng.random() < 0.3:
            a = np.round(a, 1)  # ties
        K = int(rng.integers(1, 9))
        for pol in ("greedy", "auto"):
            assert schedule("or", a, beta, K, pol)[1:] == schedule("ref", a, beta, K, pol)[1:]


def test_ffn_oracle_matches_numpy():
    """The FFN oracle (unpinned by the reference) against an independent numpy
    statement of the same math, so a typo in oracle.c cannot define parity."""
    from math import erf
    rng = np.random.default_rng(3)
    n, d, f = 5, 16, 24
    x = rng.standard_normal((n, d)).astype(np.float32)
    wi = rng.standard_normal((f, d)).astype(np.float32) / 4
    wo = rng.standard_normal((d, f)).astype(np.float32) / 5
    y = np.zeros((n, d), np.float32)
    O.or_expert_ffn(ptr(x), n, d, f, ptr(wi), ptr(wo), 0, ptr(y))
    h = x.astype(np.float64) @ wi.astype(np.float64).T
    g = 0.5 * h * (1 + np.vectorize(erf)(h / np.sqrt(2)))
    ref = g @ wo.astype(np.float64).T
    np.testing.assert_allclose(y, ref.astype(np.float32), rtol=1e-6, atol=1e-6)
