"""The library's timeline audit (infmoe_replay_check) against the reference's
replay_check (verification.hpp:108-198) on simulator outputs and on
hand-corrupted traces, plus the Chrome-trace / CSV export."""
import ctypes as C
import json

import numpy as np
import pytest

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import trace
from oracle_lib import REF, EventRec, f64a, i32a, ptr


def _ref_kinds(events, cv, K):
    ev = (EventRec * len(events))()
    for i, (st, l, e, a, b) in enumerate(events):
        ev[i] = EventRec(st, l, e, a, b)
    kinds = np.zeros(6, np.int32)
    REF.ref_replay_check(ev, len(events), ptr(f64a(cv.alphas)), cv.size(), cv.beta, K,
                         ptr(kinds))
    return {k: int(v) for k, v in zip(im.VIOLATION_KINDS, kinds) if v}


def test_clean_simulations_have_no_violations():
    rng = np.random.default_rng(5)
    for _ in range(300):
        T = int(rng.integers(1, 20))
        cv = im.CostVector(rng.uniform(0, 3, T), 1.0)
        K = int(rng.integers(1, 6))
        events, rep = im.simulate(im.auto_order(cv, K).order, cv, K)
        assert im.replay_check(events, [cv], K) == {}


@pytest.mark.skipif(REF is None, reason="compiled reference not present")
def test_injected_faults_match_reference():
    rng = np.random.default_rng(6)
    for trial in range(200):
        T = int(rng.integers(2, 10))
        cv = im.CostVector(rng.uniform(0.1, 3, T), 1.0)
        K = int(rng.integers(1, 4))
        events, _ = im.simulate(im.greedy_order(cv, K).order, cv, K)
        ev = [list(e) for e in events]
        i = int(rng.integers(0, len(ev)))
        kind = trial % 4
        if kind == 0:    # compute before its load ends
            comp = [j for j, e in enumerate(ev) if e[0] == 1][int(rng.integers(0, T))]
            ev[comp][3] -= 5.0
            ev[comp][4] -= 5.0
        elif kind == 1:  # stretch an event (duration + overlap)
            ev[i][4] += 0.7
        elif kind == 2:  # K+1 residents: every load finished at t=0
            for e in ev:
                if e[0] == 0:
                    e[3], e[4] = -1.0, 0.0
        else:            # malformed
            ev[i][3], ev[i][4] = 2.0, 1.0
        ev = [tuple(e) for e in ev]
        assert im.replay_check(ev, [cv], K) == _ref_kinds(ev, cv, K), (kind, ev)


def test_measured_mode_tolerance_and_skipped_experts():
    cv = im.CostVector(np.asarray([1.0, 2.0, 0.0]), 1.0)
    # measured-like: durations off by 1%, compute starts 1 us after load end
    ev = [(0, 0, 0, 0.0, 1.01), (1, 0, 0, 1.011, 2.02), (0, 0, 1, 1.01, 2.02),
          (1, 0, 1, 2.021, 4.04)]  # expert 2 skipped (no rows): neither loaded nor run
    assert im.replay_check(ev, [cv], 2, check_durations=False, tol_s=1e-6) == {}
    assert im.replay_check(ev, [cv], 2, check_durations=True, tol_s=1e-6)["duration_mismatch"] > 0
    assert im.replay_check(ev[:3], [cv], 2, check_durations=False)["causality"] == 1


def test_trace_export_roundtrip(tmp_path):
    cv = im.CostVector(np.asarray([0.5, 2, 1, 0.5]), 1.0)
    events, _ = im.simulate([2, 1, 0, 3], cv, 2)
    prefix = str(tmp_path / "fig3")
    trace.write(events, prefix)
    tr = json.load(open(prefix + ".trace.json"))
    xs = [e for e in tr["traceEvents"] if e["ph"] == "X"]
    assert len(xs) == 8 and {e["tid"] for e in xs} == {0, 1}
    csv = open(prefix + ".csv").read().splitlines()
    assert csv[0] == "stream,layer,expert,start_s,end_s" and len(csv) == 9
    assert csv[1].startswith("load,0,2,0.000000000,1.000000000")
