"""The PEER expert-parallel transport across PROCESSES: P = 2 or 4 ranks are P
processes on one GPU, so every peer buffer (received rows, return addresses,
results, counts, barrier flags) is a real CUDA-IPC mapping (cudaIpcGetMemHandle
/ cudaIpcOpenMemHandle in Layer::peer_setup), exchanged through the
process-shared stand-in collectives of tests/loopback_nccl/ipc_nccl.cpp (host
barriers in /dev/shm: no kernel waits on another process's kernel; the layer's
barriers use its NCCL path, INFMOE_EP_BARRIER=nccl).  The ranks' slices of
the output must equal the one-GPU layer on the whole batch bit for bit."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "loopback_nccl" / "ipc_nccl.cpp"

INPUTS = r'''
import sys, numpy as np, torch
sys.path.insert(0, "{root}")
import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
cuda = torch.device("cuda:0")
k, gate, offloaded = {k}, "{gate}", {offloaded}
N, d, f, E, P = 768, 256, 384, 8, {P}
g = torch.Generator().manual_seed(3)
x = torch.randn(N, d, generator=g).to(torch.bfloat16).to(cuda)
wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16)
wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16)
gw = (np.random.default_rng(2).standard_normal((E, d)) / d ** 0.5).astype(np.float32)
kw = dict(gate=gate, gate_weight=gw, lsh_seed=13, lsh_bits=3, max_tokens=N)
'''

RANK = INPUTS + r'''
r = int(sys.argv[1])
comm = im.ep_comm_init(bytes.fromhex("{uid}"), P, r)
El, n = E // P, N // P
wi_r, wo_r = wi[r * El:(r + 1) * El].contiguous(), wo[r * El:(r + 1) * El].contiguous()
w = (wi_r.pin_memory(), wo_r.pin_memory()) if offloaded else (wi_r.to(cuda), wo_r.to(cuda))
lay = dv.MoELayer(d, f, E, k, *w, offloaded=offloaded, K=2, ep_size=P, ep_rank=r,
                  ep_comm=comm, ep_transport="peer", **kw)
for _ in range(2):
    y, info = lay.forward(x[r * n:(r + 1) * n])
torch.cuda.synchronize()
torch.save({{"y": y.cpu(), "rows": info["local_rows"]}}, "{out}/rank%d.pt" % r)
lay.close()
im.ep_comm_destroy(comm)
print("rank ok", r)
'''

REF = INPUTS + r'''
ref = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), **kw)
y_ref, info = ref.forward(x)
torch.cuda.synchronize()
parts = [torch.load("{out}/rank%d.pt" % r, weights_only=False) for r in range(P)]
y = torch.cat([p["y"] for p in parts])
assert torch.equal(y.view(torch.int16), y_ref.cpu().view(torch.int16))
assert np.array_equal(np.concatenate([p["rows"] for p in parts]), info["counts"])
print("ok")
'''


@pytest.fixture(scope="module")
def ipc_lib(tmp_path_factory):
    so = tmp_path_factory.mktemp("ipc") / "libipc_nccl.so"
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I/usr/local/cuda/include",
                        "-o", str(so), str(SRC), "-L/usr/local/cuda/lib64", "-lcudart", "-lrt"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return so


@pytest.mark.parametrize("P,k,gate,offloaded", [(2, 1, "lsh", False), (2, 2, "softmax", False),
                                                (2, 1, "lsh", True), (4, 2, "softmax", False),
                                                (4, 1, "lsh", True)])
def test_peer_transport_across_processes(ipc_lib, tmp_path, P, k, gate, offloaded):
    uid = os.urandom(128).hex()
    env = dict(os.environ, INFMOE_NCCL_LIB=str(ipc_lib), INFMOE_EP_BARRIER="nccl")
    code = RANK.format(root=ROOT, P=P, k=k, gate=gate, offloaded=offloaded, uid=uid,
                       out=tmp_path)
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(P)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=240))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0 and "rank ok" in o, o[-2000:] + e[-4000:]
    r = subprocess.run([sys.executable, "-c", REF.format(root=ROOT, P=P, k=k, gate=gate,
                                                         offloaded=offloaded, out=tmp_path)],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
