"""The layer's own expert-parallel code path (count exchange, exchange plan,
dispatch all-to-allv, local expert FFN, combine all-to-allv, combine) with
P = 2 and 4 ranks on ONE GPU: each rank is a host thread with its own stream
and its own infmoe_layer (ep_size = P), and the transport is
tests/loopback_nccl (ncclSend/ncclRecv as stream-ordered device copies
matched on the host; no kernel waits on another rank).  The concatenated
per-rank outputs must equal the one-GPU layer on the whole batch bit for bit,
resident and offloaded, top-1 LSH and top-2 softmax, over both transports:
NCCL (grouped send/recv, host-planned) and PEER (rows pushed into the owners'
buffers, device-side plan, results written back by the FFN epilogue; the
ranks share a process, so peer buffers are plain device pointers).  Runs in a subprocess
because INFMOE_NCCL_LIB is read when NCCL is first bound."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "loopback_nccl" / "loopback_nccl.cpp"

SCRIPT = r'''
import sys, threading, numpy as np, torch
sys.path.insert(0, "{root}")
import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
cuda = torch.device("cuda:0")
P, k, gate, offloaded, transport, codec = {P}, {k}, "{gate}", {offloaded}, "{transport}", "{codec}"
N, d, f, E = 1024, 256, 384, 16
g = torch.Generator().manual_seed(7)
x = torch.randn(N, d, generator=g).to(torch.bfloat16).to(cuda)
wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16)
wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16)
gw = (np.random.default_rng(1).standard_normal((E, d)) / d ** 0.5).astype(np.float32)
kw = dict(gate=gate, gate_weight=gw, lsh_seed=11, lsh_bits=4, max_tokens=N)
ref = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), **kw)
y_ref, info_ref = ref.forward(x)
torch.cuda.synchronize()
uid = im.ep_unique_id()
El, n = E // P, N // P
ys, errs, counts = [None] * P, [], [None] * P
def rank(r):
    try:
        torch.cuda.set_device(0)
        comm = im.ep_comm_init(uid, P, r)
        wi_r, wo_r = wi[r * El:(r + 1) * El], wo[r * El:(r + 1) * El]
        w = (wi_r.contiguous().pin_memory(), wo_r.contiguous().pin_memory()) if offloaded \
            else (wi_r.to(cuda), wo_r.to(cuda))
        lay = dv.MoELayer(d, f, E, k, *w, offloaded=offloaded, K=2, ep_size=P, ep_rank=r,
                          ep_comm=comm, ep_transport=transport, h2d_codec=codec, **kw)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):  # twice: buffers are reused across forwards
                y, info = lay.forward(x[r * n:(r + 1) * n])
        s.synchronize()
        ys[r], counts[r] = y, info["local_rows"]
        lay.close()
        im.ep_comm_destroy(comm)
    except Exception as e:  # noqa: BLE001
        errs.append(repr(e))
th = [threading.Thread(target=rank, args=(r,)) for r in range(P)]
for t in th: t.start()
for t in th: t.join(timeout=120)
assert not errs, errs
assert all(not t.is_alive() for t in th), "a rank hung"
y = torch.cat(ys)
assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16)), float((y.float() - y_ref.float()).abs().max())
# every rank computed exactly the rows routed to its experts
tot = info_ref["counts"]
assert np.array_equal(np.concatenate(counts), tot), (np.concatenate(counts), tot)
print("ok")
'''


@pytest.fixture(scope="module")
def loopback_lib(tmp_path_factory):
    so = tmp_path_factory.mktemp("nccl") / "libloopback_nccl.so"
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-I/usr/local/cuda/include",
                        "-o", str(so), str(SRC), "-L/usr/local/cuda/lib64", "-lcudart"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return so


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("P,k,gate", [(2, 1, "lsh"), (4, 2, "softmax")])
@pytest.mark.parametrize("offloaded,codec", [(False, "raw"), (True, "raw"), (True, "exph")])
def test_layer_ep_ranks_as_threads_equal_single_gpu(loopback_lib, P, k, gate, offloaded, codec,
                                                    transport):
    env = dict(os.environ, INFMOE_NCCL_LIB=str(loopback_lib))
    code = SCRIPT.format(root=ROOT, P=P, k=k, gate=gate, offloaded=offloaded, transport=transport,
                         codec=codec)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("P,k,gate,offloaded", [(2, 1, "lsh", False), (4, 2, "softmax", False),
                                                (2, 1, "lsh", True)])
def test_peer_device_flag_barrier(loopback_lib, P, k, gate, offloaded):
    """The PEER transport's device-side epoch-flag barrier (ep_flag_barrier_kernel,
    the default when ranks are separate processes): here forced on for ranks as
    threads (INFMOE_EP_BARRIER=device), with every kernel module loaded up front
    (CUDA_MODULE_LOADING=EAGER) so no first launch can wait behind a spinning
    barrier; the barrier traps after 20 s rather than hang.  No collective runs
    per layer; outputs equal the one-GPU layer bit for bit."""
    env = dict(os.environ, INFMOE_NCCL_LIB=str(loopback_lib), INFMOE_EP_BARRIER="device",
               CUDA_MODULE_LOADING="EAGER", INFMOE_EP_BARRIER_TIMEOUT_S="20")
    code = SCRIPT.format(root=ROOT, P=P, k=k, gate=gate, offloaded=offloaded, transport="peer",
                         codec="raw")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
