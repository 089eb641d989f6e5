"""`bench.py --impl reference` (the driver's reference arm) runs on the host
alone and prints one JSON line with the contract's keys (CPU, no GPU)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_contract_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--cpu-sample", "8", "--steps", "1", "--warmup", "0",
                        "--host-sets", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0 and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    # the CPU path alone: the reference build and the oracle port, never the product
    libs = line["native_libs_loaded"]
    assert not any("libinfmoe" in p for p in libs), libs
    assert "oracle/_ref/libmoesim_ref.so" in libs and "oracle/liboracle.so" in libs
    assert line["config"]["layers"] == 24 and line["dtype"] == "bf16"


def test_reference_arm_nonzero_rank_exits_quietly():
    env = {"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1", "PATH": "/usr/bin:/bin"}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode == 0 and r.stdout.strip() == "", r.stderr[-2000:]
