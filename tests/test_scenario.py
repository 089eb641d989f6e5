"""The scenario front door: infmoe_scenario_resolve against the
reference's parse_scenario + to_json (scenario.hpp:188-406, compiled in place in
oracle/_ref) on valid and invalid documents -- same resolved bytes, same error
class and message; MOE_SIM_PRESETS; and the `infmoe` CLI: run / sweep
artefacts, byte-identical reruns, the SPEC examples
 and the exit codes."""
import csv
import ctypes as C
import json
import os
import subprocess
from pathlib import Path

import pytest

import paper_2106_10715_b200 as im
from oracle_lib import REF

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2106_10715_b200" / "_lib" / "infmoe"

if REF is not None:
    REF.ref_scenario_resolve.argtypes = [C.c_char_p, C.c_char_p, C.c_ulonglong]


def ours(text: str):
    n = C.c_uint64(0)
    rc = im._lib.infmoe_scenario_resolve(text.encode(), None, 0, C.byref(n))
    if rc != 0:
        return rc, im._lib.infmoe_last_error().decode()
    buf = C.create_string_buffer(n.value)
    assert im._lib.infmoe_scenario_resolve(text.encode(), buf, n.value, C.byref(n)) == 0
    return 0, buf.value.decode()


def ref(text: str):
    buf = C.create_string_buffer(1 << 20)
    rc = REF.ref_scenario_resolve(text.encode(), buf, 1 << 20)
    return rc, buf.value.decode()


HW = {"peak_flops": 1.6e15, "h2d_bandwidth": 5.5e10, "device_memory": 192 << 30,
      "reserved_memory": 8 << 30}
BASE = {"name": "c3", "seed": 7, "geometry": "cpm2", "hardware": HW,
        "workload": {"kind": "zipf", "total_tokens": 4096, "zipf_s": 1.2}, "K": 4,
        "policies": ["greedy", "naive", "serial"]}


def variant(**kw):
    d = json.loads(json.dumps(BASE))
    for k, v in kw.items():
        if v is None:
            d.pop(k, None)
        else:
            d[k] = v
    return json.dumps(d)


DOCS = {
    "base": variant(),
    "auto_K": variant(K="auto"),
    "no_K": variant(K=None),
    "geometry_object": variant(geometry={"n_layers": 2, "n_heads": 8, "d_head": 64,
                                         "d_model": 512, "d_ff": 2048,
                                         "n_experts_per_layer": 8, "bytes_per_param": 2},
                               geometry_preset="mine"),
    "cpm_small": variant(geometry="cpm-small"),
    "gating": variant(workload={"kind": "gating", "total_tokens": 512, "n_hash_bits": 6}),
    "explicit": variant(workload={"kind": "explicit", "counts": [3, 0, 9]}),
    "csv": variant(workload={"kind": "csv", "csv_path": "/tmp/w.csv"}),
    "balanced_extra_key_ok": variant(workload={"kind": "balanced", "total_tokens": 64,
                                               "zipf_s": 3}),
    "costs": json.dumps({"costs": {"alphas": [0.5, 2, 1, 0.5], "beta": 1}, "K": 2,
                         "policies": ["greedy", "exact"], "seed": 1}),
    "all_flags": variant(n_moe_layers=3, continuous_load_stream=True, skip_empty_experts=True,
                         event_overhead_s=1e-5, output_dir="/tmp/x"),
    # errors
    "unknown_top": variant(bogus=1),
    "unknown_geometry_field": variant(geometry={"n_layers": 2, "n_heads": 8, "d_head": 64,
                                                "d_model": 512, "d_ff": 2048, "x": 1,
                                                "n_experts_per_layer": 8,
                                                "bytes_per_param": 2}),
    "missing_bytes": variant(geometry={"n_layers": 2, "n_heads": 8, "d_head": 64,
                                       "d_model": 512, "d_ff": 2048,
                                       "n_experts_per_layer": 8}),
    "unknown_preset": variant(geometry="gpt5"),
    "geometry_number": variant(geometry=5),
    "bad_type": variant(geometry={"n_layers": "two", "n_heads": 8, "d_head": 64,
                                  "d_model": 512, "d_ff": 2048, "n_experts_per_layer": 8,
                                  "bytes_per_param": 2}),
    "zero_dim": variant(geometry={"n_layers": 2, "n_heads": 8, "d_head": 64, "d_model": 0,
                                  "d_ff": 2048, "n_experts_per_layer": 8,
                                  "bytes_per_param": 2}),
    "hw_reserved": variant(hardware={"peak_flops": 1e15, "h2d_bandwidth": 1e10,
                                     "device_memory": 10, "reserved_memory": 10}),
    "hw_unknown": variant(hardware=dict(HW, pcie=5)),
    "bad_kind": variant(workload={"kind": "poisson", "total_tokens": 5}),
    "zipf_s_zero": variant(workload={"kind": "zipf", "total_tokens": 5, "zipf_s": 0}),
    "explicit_empty": variant(workload={"kind": "explicit", "counts": []}),
    "missing_tokens": variant(workload={"kind": "uniform"}),
    "costs_and_workload": json.dumps({"costs": {"alphas": [1], "beta": 1},
                                      "workload": {"kind": "balanced", "total_tokens": 1},
                                      "K": 1, "policies": ["greedy"]}),
    "costs_no_K": json.dumps({"costs": {"alphas": [1], "beta": 1}, "policies": ["greedy"]}),
    "costs_negative": json.dumps({"costs": {"alphas": [-1], "beta": 1}, "K": 1,
                                  "policies": ["greedy"]}),
    "K_zero": variant(K=0),
    "K_string": variant(K="many"),
    "K_float": variant(K=2.5),
    "no_policies": variant(policies=[]),
    "missing_policies": variant(policies=None),
    "bad_policy": variant(policies=["fastest"]),
    "missing_hardware": variant(hardware=None),
    "empty_name": variant(name=""),
    "layers_zero": variant(n_moe_layers=0),
    "negative_overhead": variant(event_overhead_s=-1),
    "not_object": "[1, 2]",
}


@pytest.mark.skipif(REF is None, reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("name", sorted(DOCS))
def test_resolve_matches_reference(name):
    a, b = ours(DOCS[name]), ref(DOCS[name])
    assert a == b, (a, b)


@pytest.mark.skipif(REF is None, reason="reference build (oracle/_ref) not present")
def test_moe_sim_presets_dir(tmp_path, monkeypatch):
    (tmp_path / "tiny.json").write_text(json.dumps(
        {"n_layers": 3, "n_heads": 4, "d_head": 32, "d_model": 128, "d_ff": 512,
         "n_experts_per_layer": 4, "bytes_per_param": 2}))
    (tmp_path / "cpm2.json").write_text(json.dumps(  # shadows the builtin
        {"n_layers": 1, "n_heads": 4, "d_head": 32, "d_model": 128, "d_ff": 256,
         "n_experts_per_layer": 2, "bytes_per_param": 4}))
    monkeypatch.setenv("MOE_SIM_PRESETS", str(tmp_path))
    for g in ("tiny", "cpm2"):
        doc = variant(geometry=g)
        assert ours(doc) == ref(doc)
        assert json.loads(ours(doc)[1])["geometry_preset"] == g
    monkeypatch.setenv("MOE_SIM_PRESETS", str(tmp_path / "nope"))
    assert ours(variant())[0] == ref(variant())[0] == 2


def test_resolved_round_trip_and_seed():
    rc, text = ours(variant(seed=None))
    assert rc == 0
    seed = json.loads(text)["seed"]  # resolved from entropy, then explicit
    rc2, text2 = ours(text)
    assert rc2 == 0 and text2 == text and json.loads(text2)["seed"] == seed


def _cli(*args, env=None):
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True,
                          timeout=300, env=env)


def _write(tmp_path, doc, name="s.json"):
    p = tmp_path / name
    p.write_text(doc if isinstance(doc, str) else json.dumps(doc))
    return p


def test_cli_run_artifacts_reproducible(tmp_path):
    doc = json.loads(variant(n_moe_layers=3))
    doc["workload"] = {"kind": "gating", "total_tokens": 2048, "n_hash_bits": 5}
    cfg = _write(tmp_path, doc)
    outs = []
    for i in range(2):
        out = tmp_path / f"run{i}"
        r = _cli("run", cfg, "--out", out)
        assert r.returncode == 0, r.stderr
        outs.append(out)
    files = sorted(p.relative_to(outs[0]) for p in outs[0].rglob("*") if p.is_file())
    assert {str(f) for f in files} >= {"summary.csv", "resolved.json", "meta.json",
                                       "greedy/trace.json", "greedy/events.csv",
                                       "greedy/report.json", "serial/report.json"}
    for f in files:
        if f.name != "meta.json":
            assert (outs[0] / f).read_bytes() == (outs[1] / f).read_bytes(), f
    rows = {r["policy"]: r for r in csv.DictReader(open(outs[0] / "summary.csv"))}
    assert float(rows["greedy"]["makespan_s"]) <= float(rows["serial"]["makespan_s"])
    trace = json.loads((outs[0] / "greedy" / "trace.json").read_text())
    names = {e["args"]["name"] for e in trace["traceEvents"] if e["ph"] == "M"}
    assert names == {"load", "compute"}
    ev = list(csv.DictReader(open(outs[0] / "greedy" / "events.csv")))
    assert len(ev) == 2 * 3 * 32 and set(ev[0]) == {"stream", "layer", "expert", "start_s",
                                                    "end_s"}
    rep = json.loads((outs[0] / "greedy" / "report.json").read_text())
    assert len(rep["per_layer"]) == 3 and rep["K"] == 4
    # the resolved scenario re-runs to the same artefacts
    r = _cli("run", outs[0] / "resolved.json", "--out", tmp_path / "rerun")
    assert r.returncode == 0
    assert (tmp_path / "rerun" / "greedy" / "events.csv").read_bytes() == \
        (outs[0] / "greedy" / "events.csv").read_bytes()


def test_cli_spec_examples(tmp_path):
    # Figure 3 instance, naive policy: compute_stall > 0
    cfg = _write(tmp_path, {"costs": {"alphas": [0.5, 2, 1, 0.5], "beta": 1}, "K": 2,
                            "policies": ["naive", "greedy"], "seed": 1})
    r = _cli("run", cfg, "--out", tmp_path / "fig3")
    assert r.returncode == 0, r.stderr
    rows = {x["policy"]: x for x in csv.DictReader(open(tmp_path / "fig3" / "summary.csv"))}
    assert float(rows["naive"]["compute_stall_s"]) == 0.5
    assert float(rows["greedy"]["makespan_s"]) == 5.0
    # empty policy set -> exit 2; K < 1 -> exit 3
    assert _cli("run", _write(tmp_path, variant(policies=[]), "e.json")).returncode == 2
    assert _cli("run", _write(tmp_path, variant(K=0), "k.json")).returncode == 3
    assert _cli("run", tmp_path / "missing.json").returncode == 2


def test_cli_sweeps(tmp_path):
    cfg = _write(tmp_path, variant(policies=["greedy"], workload={"kind": "balanced",
                                                                    "total_tokens": 1 << 20}))
    # K over [1..8]: greedy makespan non-increasing
    r = _cli("sweep", cfg, "--axis", "K", "--values", "1,2,3,4,5,6,7,8", "--jobs", "4",
             "--out", tmp_path / "k")
    assert r.returncode == 0, r.stderr
    ms = [float(x["makespan_s"]) for x in csv.DictReader(open(tmp_path / "k" / "sweep.csv"))]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(ms, ms[1:]))
    # bandwidth x2 -> beta halves exactly
    r = _cli("sweep", cfg, "--axis", "bandwidth", "--values", "2.5e10,5e10", "--out",
             tmp_path / "bw")
    rows = list(csv.DictReader(open(tmp_path / "bw" / "sweep.csv")))
    assert float(rows[0]["beta_s"]) == 2 * float(rows[1]["beta_s"])
    # total_tokens x2 under balanced -> all alpha double, beta constant
    r = _cli("sweep", cfg, "--axis", "total_tokens", "--values", "4096,8192", "--out",
             tmp_path / "tt")
    rows = list(csv.DictReader(open(tmp_path / "tt" / "sweep.csv")))
    assert float(rows[1]["sum_alpha_s"]) == 2 * float(rows[0]["sum_alpha_s"])
    assert rows[0]["beta_s"] == rows[1]["beta_s"]
    # rows do not depend on --jobs
    r1 = _cli("sweep", cfg, "--axis", "K", "--values", "3,1,2", "--jobs", "1", "--out",
              tmp_path / "j1")
    r3 = _cli("sweep", cfg, "--axis", "K", "--values", "3,1,2", "--jobs", "3", "--out",
              tmp_path / "j3")
    assert r1.stdout == r3.stdout and r1.returncode == 0
    # an axis the scenario cannot take -> exit 2
    assert _cli("sweep", cfg, "--axis", "zipf_s", "--values", "1.1").returncode == 2
    assert _cli("sweep", cfg, "--axis", "colour", "--values", "1").returncode == 2


def test_cli_seed_override_and_resolve(tmp_path):
    cfg = _write(tmp_path, variant())
    r = _cli("resolve", cfg)
    assert r.returncode == 0 and json.loads(r.stdout)["seed"] == 7
    a = _cli("run", cfg, "--seed", "11", "--out", tmp_path / "a")
    b = _cli("run", cfg, "--seed", "12", "--out", tmp_path / "b")
    assert a.returncode == b.returncode == 0
    assert json.loads((tmp_path / "a" / "resolved.json").read_text())["seed"] == 11
    assert (tmp_path / "a" / "greedy" / "events.csv").read_bytes() != \
        (tmp_path / "b" / "greedy" / "events.csv").read_bytes()


def test_cpp_scenario_wrappers(tmp_path):
    """The same front door from C++ through include/infmoe/moesim.hpp."""
    exe = tmp_path / "scenario_demo"
    lib_dir = Path(im.library_path()).parent
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", str(ROOT / "tests" / "cpp" /
                                                             "scenario_demo.cpp"),
                    f"-I{ROOT / 'include'}", f"-L{lib_dir}", "-linfmoe",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True, capture_output=True)
    cfg = _write(tmp_path, variant(policies=["greedy", "serial"]))
    r = subprocess.run([str(exe), str(cfg), str(tmp_path / "o")], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    summary, table, verdict = r.stdout.split("---\n")
    assert summary.startswith("policy,makespan_s") and "greedy," in summary
    rows = table.strip().splitlines()
    assert len(rows) == 1 + 3 * 2 and all(r.startswith("K,") for r in rows[1:])  # 3 K x 2 policies
    assert verdict.strip() == "ok"
    assert (tmp_path / "o" / "run" / "greedy" / "events.csv").exists()
    assert (tmp_path / "o" / "sweep" / "sweep.csv").exists()
