"""The LSH gate's certified fast path (sign of a parallel fp64 dot with an error
bound, exact sequential chain only when ambiguous) must give exactly the
reference's codes: gating.hpp:70-80 accumulates dot += x*w left to right with
separate roundings, and a bit is dot >= 0.

Cases that defeat a naive parallel sign are built in on purpose: hyperplanes
whose exact dot is +-1e-20 while the sequential double sum is exactly +0, an
exact cancellation, all-zero / -0 rows, NaN and Inf rows.  Expected codes come
from a pure-Python left-to-right loop (CPython floats: IEEE binary64, no
contraction) for the crafted rows, and from the reference's lsh_codes for the
random rows.  Each path (the fp64-MMA fast kernel, the DFMA fast kernel, each
with its exact chain forced, and the all-sequential ring kernel) runs in its
own subprocess because the mode is read once per process.
"""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, "{root}")
from paper_2106_10715_b200 import device as dv
d = np.load("{inp}")
x = torch.from_numpy(d["x"]).to("cuda")
if d["bf16"]:
    x = x.to(torch.bfloat16)
proj = torch.from_numpy(d["proj"]).to("cuda")
codes, idx, w, cnt = dv.gate_lsh(x, proj, int(d["E"]))
torch.cuda.synchronize()
np.save("{out}", codes.cpu().numpy().view(np.uint32))
print("ok")
'''


def _seq_code(xrow, proj):
    code = 0
    for j in range(proj.shape[0]):
        dot = 0.0
        for a, b in zip(xrow.tolist(), proj[j].tolist()):
            dot = dot + a * b
        if dot >= 0.0:
            code |= 1 << j
    return code


def _case(bf16: bool):
    rng = np.random.default_rng(3)
    N, d, bits, E = 64, 64, 3, 8
    proj = rng.standard_normal((bits, d))
    proj[:, :3] = [[1.0, -1.0, 0.0],      # exact cancellation: dot == +0
                   [1.0, 1e-20, -1.0],    # exact +1e-20, sequential +0
                   [1.0, -1e-20, -1.0]]   # exact -1e-20, sequential +0 (naive sign: 0)
    x = rng.standard_normal((N, d)).astype(np.float32)
    x[0, :] = 0.0
    x[0, :3] = 1.0                        # the crafted rows: only the first 3 columns
    x[1, :] = 0.0
    x[1, :3] = [2.0, 2.0, 2.0]
    x[2, :] = 0.0                         # all-zero row
    x[3, :] = -0.0                        # negative zeros
    x[4, 5] = np.nan
    x[5, 7] = np.inf
    x[6, 9] = -np.inf
    x[7, :] *= 1e-30                      # tiny but nonzero
    if bf16:  # the values the kernel sees
        import torch
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    expect = np.array([_seq_code(x[t].astype(np.float64), proj) for t in range(N)], np.uint32)
    return x, proj, E, expect


@pytest.mark.parametrize("bf16", [True, False])
@pytest.mark.parametrize("mode", [{}, {"INFMOE_LSH_FORCE_EXACT": "1"}, {"INFMOE_LSH_MMA": "0"},
                                  {"INFMOE_LSH_MMA": "0", "INFMOE_LSH_FORCE_EXACT": "1"},
                                  {"INFMOE_LSH_FAST": "0"}])
def test_lsh_paths_match_sequential_reference(tmp_path, bf16, mode):
    x, proj, E, expect = _case(bf16)
    inp = tmp_path / "in.npz"
    np.savez(inp, x=x, proj=np.ascontiguousarray(proj), E=E, bf16=bf16)
    out = tmp_path / "codes.npy"
    env = dict(os.environ, **mode)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, inp=inp, out=out)],
                       env=env, capture_output=True, text=True, timeout=180)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
    got = np.load(out)
    bad = np.nonzero(got != expect)[0]
    assert bad.size == 0, [(int(t), int(got[t]), int(expect[t])) for t in bad[:8]]
    # the crafted rows decide bits 1 and 2 against the exact sign
    assert expect[0] & 0b111 == 0b111 and expect[1] & 0b111 == 0b111
