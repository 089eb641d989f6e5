"""The cta_group::2 (2-SM) variant of the fused expert FFN, selected with
INFMOE_FFN_PAIR=1, must equal the one-SM kernel bit for bit, and the banded
tile order for experts spanning many token chunks (INFMOE_FFN_BAND_MB) must
equal the plain chunk-fastest order.  Each case runs
in a fresh subprocess (the mode is read once per process) under a timeout."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, "{root}")
from paper_2106_10715_b200 import device as dv
cuda = torch.device("cuda:0")
counts = {counts}
E, d, f = len(counts), {d}, {f}
R = int(sum(counts))
offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=cuda)
g = torch.Generator(device="cpu").manual_seed(5)
x = torch.randn(R, d, generator=g).to(torch.bfloat16).to(cuda)
wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(cuda)
wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(cuda)
h, y = dv.expert_ffn_fused(x, offs, wi, wo)
torch.cuda.synchronize()
torch.save({{"h": h.cpu(), "y": y.cpu()}}, "{out}")
print("ok")
'''


def _run(pair: bool, counts, d, f, out, **knobs):
    env = dict(os.environ, INFMOE_FFN_PAIR="1" if pair else "0", **knobs)
    code = SCRIPT.format(root=ROOT, counts=counts, d=d, f=f, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("counts,d,f", [([128, 0, 1, 300, 127, 129, 256, 513], 256, 512),
                                        ([150] * 16, 512, 1024)])
def test_pair_kernel_equals_single(tmp_path, counts, d, f):
    import torch
    a, b = str(tmp_path / "pair.pt"), str(tmp_path / "single.pt")
    _run(True, counts, d, f, a)
    _run(False, counts, d, f, b)
    pa, pb = torch.load(a), torch.load(b)
    assert torch.equal(pa["h"].view(torch.int16), pb["h"].view(torch.int16))
    assert torch.equal(pa["y"].view(torch.int16), pb["y"].view(torch.int16))


@pytest.mark.parametrize("pair", [True, False])
def test_banded_tile_order_is_bit_identical(tmp_path, pair):
    """A 1 MB band budget at d=512/f=1024 gives bands of 5 (phase 1) and 2
    (phase 2) chunks of 192 rows, so the 2500- and 1300-row experts run in
    several bands with a narrower last one; forced L2 policies change nothing
    either.  Everything must equal one band per expert (the previous order)."""
    import torch
    counts, d, f = [2500, 0, 700, 33, 1300], 512, 1024
    ref = str(tmp_path / "ref.pt")
    _run(pair, counts, d, f, ref, INFMOE_FFN_BAND_MB="0", INFMOE_FFN_POLICY="02")
    r = torch.load(ref)
    for i, knobs in enumerate([dict(INFMOE_FFN_BAND_MB="1"),
                               dict(INFMOE_FFN_BAND_MB="1", INFMOE_FFN_POLICY="11"),
                               dict(INFMOE_FFN_BAND_MB="3", INFMOE_FFN_POLICY="22")]):
        out = str(tmp_path / f"band{i}.pt")
        _run(pair, counts, d, f, out, **knobs)
        o = torch.load(out)
        assert torch.equal(o["h"].view(torch.int16), r["h"].view(torch.int16)), knobs
        assert torch.equal(o["y"].view(torch.int16), r["y"].view(torch.int16)), knobs
