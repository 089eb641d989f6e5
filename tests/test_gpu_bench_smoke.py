"""bench.py end to end on one GPU in a short mode (1 warm-up + 1 timed step,
no C5 / pinned / CPU legs): the JSON line carries the contract's keys and the
packed stream is bit-identical to the raw stream."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_bench_short_run_contract():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "1",
                        "--resident-steps", "1", "--no-cpu-baseline", "--no-c5", "--pin-frac", "0"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "e2e", "h2d", "roofline",
                "resident", "gpu_launches", "clocks", "raw_stream"):
        assert key in line, key
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["h2d_codec"] == "exph"
    assert line["h2d"]["bit_identical_to_raw_stream"]
    assert line["h2d"]["replay_check_violations"] == {}
    assert line["resident"]["bit_identical_to_offloaded"]
    assert line["value"] > line["raw_stream"]["value"]  # fewer bytes over the same link
