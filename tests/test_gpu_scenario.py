"""`infmoe run --execute`: a scenario drives the real offload executor on the GPU
(SURVEY §8f-3).  For count workloads (zipf, explicit) the layers run the
scenario's own counts through infmoe_layer_forward_routed, so the MEASURED
per-layer counts and expert orders equal the simulated ones; for a gating
workload the layer's LSH gate routes the scenario's hidden states.  Every
measured timeline passes replay_check's rules with <= K residents, and the
measured artefacts sit next to the simulated ones."""
import csv
import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2106_10715_b200" / "_lib" / "infmoe"

GEOM = {"n_layers": 3, "n_heads": 8, "d_head": 64, "d_model": 512, "d_ff": 1024,
        "n_experts_per_layer": 8, "bytes_per_param": 2}
HW = {"peak_flops": 1.6e15, "h2d_bandwidth": 5.5e10, "device_memory": 192 << 30,
      "reserved_memory": 8 << 30}


@pytest.mark.parametrize("workload", [
    {"kind": "zipf", "total_tokens": 3000, "zipf_s": 1.1},
    {"kind": "explicit", "counts": [500, 0, 120, 7, 300, 0, 64, 9]},
    {"kind": "gating", "total_tokens": 2048, "n_hash_bits": 3}])
def test_execute_scenario(tmp_path, workload):
    doc = {"name": "gpu", "seed": 5, "geometry": GEOM, "hardware": HW, "workload": workload,
           "K": 2, "policies": ["greedy", "naive", "serial"], "skip_empty_experts": True}
    cfg = tmp_path / "s.json"
    cfg.write_text(json.dumps(doc))
    r = subprocess.run([str(CLI), "run", str(cfg), "--execute", "--out", str(tmp_path / "o"),
                        "--repeats", "2"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    out = tmp_path / "o"
    rows = {x["policy"]: x for x in csv.DictReader(open(out / "measured" / "summary.csv"))}
    assert set(rows) == {"greedy", "naive"}  # serial is a simulator mode only
    for pol in ("greedy", "naive"):
        m = json.loads((out / "measured" / pol / "report.json").read_text())
        s = json.loads((out / pol / "report.json").read_text())
        assert m["replay_check_violations"] == 0, m["replay_check_kinds"]
        assert m["peak_resident_experts"] <= 2
        assert m["makespan"] > 0 and 0.2 < m["measured_over_simulated"] < 50
        ev = list(csv.DictReader(open(out / "measured" / pol / "events.csv")))
        if workload["kind"] != "gating":
            # the executor ran exactly the scenario's experts in the simulated order
            for lay in range(3):
                want = [e for e in s["per_layer"][lay]["schedule"]["order"]]
                sim_ev = list(csv.DictReader(open(out / pol / "events.csv")))
                sim_loads = [int(x["expert"]) for x in sim_ev
                             if x["stream"] == "load" and int(x["layer"]) == lay]
                got = [int(x["expert"]) for x in sorted(ev, key=lambda x: float(x["start_s"]))
                       if x["stream"] == "load" and int(x["layer"]) == lay]
                assert got == sim_loads and len(want) == len(sim_loads)
