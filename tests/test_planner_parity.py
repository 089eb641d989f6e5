"""The product's planning layer (libinfmoe.so through the C-ABI) against the
reference: golden vectors frozen from moesim, and the compiled reference live
on randomised instances (T <= 64, K in [1, 8], Zipf / balanced / tied counts).
Expert orders, feasibility, diagnosis and timelines must be bit-identical."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2106_10715_b200 as im
from oracle_lib import REF, f32_to_bf16_bits, f64a, i32a, ptr, schedule

G = json.loads((Path(__file__).parent / "golden" / "moesim_reference.json").read_text())
DIAG_CODE = {None: -1, "feasible": 0, "too_little_compute": 1, "imbalanced": 2}
METH_CODE = {"greedy": 0, "exact_fallback": 1, "naive": 2}


def test_prng_and_projection_golden():
    for s, t, v in G["derive_seed"]:
        assert im.derive_seed(s, t) == v
    for s, v in G["splitmix64"].items():
        assert im.splitmix64(int(s)) == v
    assert im.gaussian_stream(0, 21).tolist() == G["gaussian_tokens_seed0_3x7"]
    p = im.gating_projection(0, 5, 768).reshape(-1)
    for i, v in G["gating_projection_seed0_5x768_sample"].items():
        assert p[int(i)] == v


def test_workloads_golden():
    kinds = {0: "uniform", 1: "zipf", 2: "balanced"}
    for w in G["workloads"]:
        c = im.synthetic_workload(kinds[w["kind"]], w["total"], w["E"], w["seed"], w["zipf_s"])
        assert c.tolist() == w["counts"]


def test_cost_model_golden():
    for d, f, b, v in G["expert_param_bytes"]:
        assert im.expert_param_bytes(im.make_geometry(d, f, 1, b)) == v
    for d, f, n, v in G["expert_flops"]:
        assert im.expert_flops(im.make_geometry(d, f, 1, 2), n) == v
    for c in G["costs"]:
        d, f, b = c["geom"]
        cv = im.compute_costs(c["counts"], im.make_geometry(d, f, len(c["counts"]), b),
                              im.Hardware(c["peak"], c["bw"], 2, 1))
        assert cv.alphas.tolist() == c["alphas"] and cv.beta == c["beta"]
    g = im.geometry_preset("cpm2")
    assert im.resident_capacity(g, im.Hardware(1e12, 16e9, 16 << 30, 8 << 30)) == 51
    with pytest.raises(im.CapacityError):
        im.resident_capacity(g, im.Hardware(1e12, 16e9, 100, 10))
    with pytest.raises(im.ConfigError):
        im.resident_capacity(g, im.Hardware(1e12, 16e9, 10, 10))


def test_schedules_golden():
    for s in G["schedules"]:
        cv = im.CostVector(np.asarray(s["alphas"], np.float64), s["beta"])
        K = s["K"]
        for name, fn in (("greedy", im.greedy_order), ("auto", im.auto_order),
                         ("naive", im.naive_order)):
            got = fn(cv, K)
            want = s[name]
            assert got.order == want["order"], (name, s)
            assert got.feasible == want["feasible"]
            assert DIAG_CODE[got.diagnosis] == want["diagnosis"]
            assert METH_CODE[got.method] == want["method"]
        if s["exact"] is not None:
            got = im.exact_order(cv, K)
            assert (got.order, got.feasible, DIAG_CODE[got.diagnosis]) == (
                s["exact"]["order"], s["exact"]["feasible"], s["exact"]["diagnosis"])
        assert DIAG_CODE[im.diagnose(cv, K)] == s["diagnose"]
        assert im.lower_bound(cv) == s["lower_bound"]
        ci = s["check_identity"]
        rep = im.check_constraints(list(range(cv.size())), cv, K)
        assert rep.feasible == ci["feasible"] and rep.slack.tolist() == ci["slack"]
        if not rep.feasible:
            assert rep.first_violation["position"] == ci["viol_pos"]
            assert (rep.first_violation["bound"] == "lower") == (ci["viol_side"] == 0)


def test_simulations_golden():
    for s in G["simulations"]:
        costs = [im.CostVector(np.asarray(a, np.float64), b) for a, b in s["layers"]]
        events, rep, orders = im.simulate_model(costs, s["K"],
                                                "overlapped" if s["mode"] == 0 else "serial",
                                                s["policy"], bool(s["continuous"]))
        assert sum(orders, []) == s["orders"]
        assert [list(e) for e in events] == s["events"]
        assert [rep.makespan, rep.compute_busy, rep.load_busy, rep.compute_stall,
                rep.peak_resident_experts, rep.overlap_efficiency] == s["report"]


def test_error_behaviour_matches_reference():
    cv = im.CostVector(np.asarray([1.0, 2.0]), 1.0)
    with pytest.raises(ValueError):
        im.check_constraints([0, 0], cv, 1)           # not a permutation: invalid_argument
    with pytest.raises(ValueError):
        im.greedy_order(cv, 0)                         # K < 1: invalid_argument
    with pytest.raises(im.ConfigError):
        im.greedy_order(im.CostVector(np.asarray([1.0]), 0.0), 1)  # beta must be > 0
    with pytest.raises(im.ConfigError):
        im.greedy_order(im.CostVector(np.asarray([-1.0]), 1.0), 1)
    with pytest.raises(ValueError):
        im.exact_order(im.CostVector(np.zeros(13), 1.0), 1)   # T > max_T: invalid_argument
    with pytest.raises(im.ConfigError):
        im.synthetic_workload("zipf", 10, 4, 0, zipf_s=0.0)
    with pytest.raises(im.ConfigError):
        im.gating_projection(0, 0, 10)
    with pytest.raises(im.CapacityError):
        im.clamp_explicit_capacity(0, 5, [])
    w = []
    assert im.clamp_explicit_capacity(9, 5, w) == 5 and w == ["K clamped from 9 to capacity 5"]
    assert im.validate_geometry(im.geometry_preset("cpm2")) == []
    assert len(im.validate_geometry(im.make_geometry(100, 10, 2, 2, n_heads=3, d_head=7))) == 1
    with pytest.raises(im.ConfigError):
        im.geometry_preset("nope")


@pytest.mark.skipif(REF is None, reason="compiled reference not present")
def test_random_instances_live_vs_reference():
    rng = np.random.default_rng(12345)
    peak, bw = 1643.6e12, 55.5e9
    for trial in range(1500):
        T = int(rng.choice([2, 5, 8, 12, 16, 32, 64]))
        K = int(rng.integers(1, 9))
        kind = trial % 4
        if kind == 0:    # PCIe regime, routed counts (too_little_compute, ties)
            counts = rng.integers(0, 400, T)
            cv = im.compute_costs(counts, im.make_geometry(4096, 10240, T, 2),
                                  im.Hardware(peak, bw, 2, 1))
        elif kind == 1:  # big batches: feasible regime
            counts = rng.zipf(1.5, T) * 20000
            cv = im.compute_costs(counts, im.make_geometry(4096, 10240, T, 2),
                                  im.Hardware(peak, bw, 2, 1))
        elif kind == 2:  # SPEC acceptance distribution
            beta = float(rng.uniform(0.1, 2))
            cv = im.CostVector(rng.uniform(0, 3 * beta, T), beta)
        else:            # heavy ties
            beta = 1.0
            cv = im.CostVector(rng.integers(0, 4, T).astype(np.float64) * 0.5, beta)
        for pol in ("greedy", "auto"):
            got = im.greedy_order(cv, K) if pol == "greedy" else im.auto_order(cv, K)
            rc, order, feas, diag, meth = schedule("ref", cv.alphas, cv.beta, K, pol)
            assert got.order == order and got.feasible == feas
            assert DIAG_CODE[got.diagnosis] == diag and METH_CODE[got.method] == meth


@pytest.mark.skipif(REF is None, reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("threads", [1, 3, 0])
def test_gaussian_fill_typed_is_the_reference_stream(threads):
    """infmoe_gaussian_fill_typed (the bench's and tests' synthetic tensors,
    SURVEY 8(d)) == the reference's gaussian_tokens (prng.hpp GaussianStream) x
    scale, rounded f32 RN -> bf16 RNE, for any thread count; one long stream
    (parallel Box-Muller over the sequential engine outputs) and many short ones."""
    for n_mats, n in ((1, 200_001), (7, 5_003)):
        seeds = [im.derive_seed(77, t) for t in range(n_mats)]
        scales = [1.0 / (t + 1.5) for t in range(n_mats)]
        outs = [np.empty(n, np.uint16) for _ in range(n_mats)]
        outs32 = [np.empty(n, np.float32) for _ in range(n_mats)]
        im.gaussian_fill_typed("bf16", seeds, scales, n, outs, threads=threads)
        im.gaussian_fill_typed("f32", seeds, scales, n, outs32, threads=threads)
        for sd, sc, o, o32 in zip(seeds, scales, outs, outs32):
            g = np.empty(n, np.float64)
            REF.ref_gaussian_tokens(sd, n, 1, ptr(g))
            v = (g * sc).astype(np.float32)
            assert np.array_equal(o32.view(np.uint32), v.view(np.uint32))
            assert np.array_equal(o, f32_to_bf16_bits(v))
