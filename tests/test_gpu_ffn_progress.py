"""Forward progress of the persistent fused expert FFN when most of the GPU is
taken by a concurrent kernel.

The FFN's phase-2 tiles of an expert wait for all of that expert's phase-1
tiles.  With tiles striped statically over the grid, CTAs that are resident
would spin on phase-1 tiles owned by CTAs that cannot be scheduled -- here the
other SMs are held by spinners that are only released AFTER the FFN (and a
second FFN on a third stream) completed, so static striding deadlocks (until
the spinners' 20 s timeout) while claiming tiles in global order from a counter
(expert_gemm.cu claim_tile) finishes on the few free SMs.  Both kernels (the
cta_group::2 pair kernel and the one-SM kernel) must also give the same bits as
an unobstructed launch.  Each case runs in a fresh subprocess under a timeout."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, "{root}")
from paper_2106_10715_b200 import device as dv
cuda = torch.device("cuda:0")
sms = torch.cuda.get_device_properties(0).multi_processor_count
E, d, f = 8, 512, 1024
counts = [150, 0, 90, 300, 128, 1, 256, 200]
R = int(sum(counts))
offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=cuda)
g = torch.Generator(device="cpu").manual_seed(7)
x = torch.randn(R, d, generator=g).to(torch.bfloat16).to(cuda)
wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(cuda)
wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(cuda)
wi2, wo2 = wi.flip(0).contiguous(), wo.flip(0).contiguous()
h_ref, y_ref = dv.expert_ffn_fused(x, offs, wi, wo)
h_ref2, y_ref2 = dv.expert_ffn_fused(x, offs, wi2, wo2)
torch.cuda.synchronize()
release = torch.zeros(1, dtype=torch.int32, device=cuda)
timed_out = torch.zeros(1, dtype=torch.int32, device=cuda)
sa, sb, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
# warm the caching allocator on both streams: no cudaMalloc (which may wait for
# the device) may happen while the spinners hold the SMs
for s_, (a_, b_) in ((sb, (wi, wo)), (sc, (wi2, wo2))):
    with torch.cuda.stream(s_):
        tmp = dv.expert_ffn_fused(x, offs, a_, b_)
    torch.cuda.synchronize()
    del tmp
# and load every kernel used below once: with CUDA lazy loading the FIRST
# launch of a kernel loads its module, which waits for running kernels
dummy = torch.zeros(1, dtype=torch.int32, device=cuda)
dv.set_flag(dummy, stream=sb)
with torch.cuda.stream(sb):
    torch.cuda._sleep(1000)
torch.cuda.synchronize()
free = {free}
dv.occupy_sms(sms - free, release, timed_out, stream=sa)
t0 = time.time()
with torch.cuda.stream(sb):
    torch.cuda._sleep(2_000_000)  # let the spinners take their SMs first
    h1, y1 = dv.expert_ffn_fused(x, offs, wi, wo)
with torch.cuda.stream(sc):
    torch.cuda._sleep(2_000_000)
    h2, y2 = dv.expert_ffn_fused(x, offs, wi2, wo2)
sb.wait_stream(sc)
dv.set_flag(release, stream=sb)  # the spinners go only once both FFNs are done
torch.cuda.synchronize()
el = time.time() - t0
assert int(timed_out.item()) == 0, "spinners timed out: the FFN needed the occupied SMs"
for a, b in ((h1, h_ref), (y1, y_ref), (h2, h_ref2), (y2, y_ref2)):
    assert torch.equal(a.view(torch.int16), b.view(torch.int16))
print("ok", round(el, 3))
'''


@pytest.mark.parametrize("pair", ["1", "0"])
@pytest.mark.parametrize("free", [4, 10])
def test_fused_ffn_completes_on_few_free_sms(pair, free):
    env = dict(os.environ, INFMOE_FFN_PAIR=pair)
    code = SCRIPT.format(root=ROOT, free=free)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=180)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
