"""Expert parallelism on the GPU (this pool has one GPU per call):
1) P virtual ranks on one device run the full EP data path through the
   product's kernels (gate, dispatch, gather, EP plan, expert FFN on the rank's
   expert shard, scatter, combine) with device copies as the transport; the
   result must equal the one-GPU layer bit for bit;
2) the layer's transports run on a real 1-rank NCCL communicator (self
   exchange), resident and offloaded, and must equal the plain layer bit for
   bit: NCCL (grouped ncclSend/ncclRecv) and PEER (all-gather of the buffer
   addresses, device-side plan, pushes, 1-int all-reduce barriers)."""
import numpy as np
import pytest
import torch

import paper_2106_10715_b200 as im
from paper_2106_10715_b200 import device as dv
from oracle_lib import fill_bf16

pytestmark = pytest.mark.gpu


def _weights(cuda, E, d, f, seed=3):
    t = lambda b, sh: torch.from_numpy(b.view(np.int16).reshape(sh)).view(torch.bfloat16)
    wi = t(fill_bf16(seed, E * f * d, 1.7320508 / d ** 0.5), (E, f, d))
    wo = t(fill_bf16(seed + 1, E * d * f, 1.534 * 1.7320508 / f ** 0.5), (E, d, f))
    x = t(fill_bf16(seed + 2, 1024 * d, 1.7320508), (1024, d)).to(cuda)
    return x, wi, wo


@pytest.mark.parametrize("P,k", [(2, 1), (4, 2)])
def test_virtual_ranks_equal_single_gpu(cuda, P, k):
    N, d, f, E = 1024, 256, 384, 16
    x, wi, wo = _weights(cuda, E, d, f)
    gw = (np.random.default_rng(1).standard_normal((E, d)) / d ** 0.5).astype(np.float32)
    ref_layer = dv.MoELayer(d, f, E, k, wi.to(cuda), wo.to(cuda), gate="softmax",
                            gate_weight=gw, max_tokens=N)
    y_ref, _ = ref_layer.forward(x)
    gwt = torch.from_numpy(gw).to(cuda)
    El, n = E // P, N // P
    ranks = []
    for r in range(P):  # route on every rank
        xs = x[r * n:(r + 1) * n]
        idx, w, cnt = dv.gate_softmax_topk(xs, gwt, k)
        off, perm, inv = dv.dispatch(idx, E)
        xp = dv.gather_rows(xs, perm, k)
        ranks.append(dict(w=w, cnt=cnt.cpu().numpy(), inv=inv, xp=xp))
    allc = np.stack([rk["cnt"] for rk in ranks])
    plans = [im.ep_plan(P, r, E, allc[r], allc[:, r * El:(r + 1) * El].reshape(-1))
             for r in range(P)]
    # dispatch all-to-allv (device copies stand in for NCCL)
    recv = [torch.empty((plans[r].n_recv, d), dtype=torch.bfloat16, device=cuda)
            for r in range(P)]
    for s in range(P):
        for r in range(P):
            a, b = plans[s].send_off[r], plans[s].send_off[r] + plans[s].send_rows[r]
            c = plans[r].recv_off[s]
            recv[r][c:c + (b - a)] = ranks[s]["xp"][a:b]
    back = []
    for r in range(P):  # expert compute on each rank's shard
        li = torch.from_numpy(plans[r].local_index).to(cuda)
        loc = dv.gather_rows(recv[r], li, 1)
        offs = torch.from_numpy(plans[r].local_offsets).to(cuda)
        _, ly = dv.expert_ffn(loc, offs, wi[r * El:(r + 1) * El].to(cuda),
                              wo[r * El:(r + 1) * El].to(cuda))
        back.append(dv.scatter_rows(ly, li, plans[r].n_recv))
    ys = []
    for s in range(P):  # combine all-to-allv + combine
        yp = torch.empty((n * k, d), dtype=torch.bfloat16, device=cuda)
        for r in range(P):
            a, b = plans[s].send_off[r], plans[s].send_off[r] + plans[s].send_rows[r]
            c = plans[r].recv_off[s]
            yp[a:b] = back[r][c:c + (b - a)]
        ys.append(dv.combine(yp, ranks[s]["inv"], ranks[s]["w"], n, k))
    y = torch.cat(ys)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16))
    ref_layer.close()


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("offloaded", [False, True])
def test_layer_nccl_transport_self_exchange(cuda, offloaded, transport):
    N, d, f, E = 512, 256, 384, 8
    x, wi, wo = _weights(cuda, E, d, f, seed=9)
    x = x[:N].contiguous()
    plain = dv.MoELayer(d, f, E, 1, wi.to(cuda), wo.to(cuda), gate="lsh", lsh_seed=3, lsh_bits=3,
                        max_tokens=N)
    y0, info0 = plain.forward(x)
    comm = im.ep_comm_init(im.ep_unique_id(), 1, 0)
    try:
        w_in = wi.pin_memory() if offloaded else wi.to(cuda)
        w_out = wo.pin_memory() if offloaded else wo.to(cuda)
        ep = dv.MoELayer(d, f, E, 1, w_in, w_out, gate="lsh", lsh_seed=3, lsh_bits=3,
                         offloaded=offloaded, K=2, max_tokens=N, ep_size=1, ep_rank=0,
                         ep_comm=comm, ep_transport=transport)
        y1, info1 = ep.forward(x)
        y2, _ = ep.forward(x)  # buffers reused
        torch.cuda.synchronize()
        assert torch.equal(y0.view(torch.int16), y1.view(torch.int16))
        assert torch.equal(y1.view(torch.int16), y2.view(torch.int16))
        ep.close()
    finally:
        im.ep_comm_destroy(comm)
    plain.close()


def test_peer_transport_resident_stack_is_graph_capturable(cuda):
    """The PEER transport plans on the device and barriers on the stream, so a
    resident expert-parallel stack has no host round trip: it is captured as
    one CUDA graph (real NCCL, 1-rank communicator) and replays bit-identical
    to eager execution."""
    N, d, f, E, L = 512, 256, 384, 8, 3
    x, wi, wo = _weights(cuda, E, d, f, seed=13)
    x = x[:N].contiguous()
    comm = im.ep_comm_init(im.ep_unique_id(), 1, 0)
    try:
        layers = [dv.MoELayer(d, f, E, 1, wi.to(cuda), wo.to(cuda), gate="lsh", lsh_seed=20 + l,
                              lsh_bits=3, max_tokens=N, ep_size=1, ep_rank=0, ep_comm=comm,
                              ep_transport="peer") for l in range(L)]
        bufs = [torch.empty_like(x) for _ in range(2)]

        def run():
            cur = x
            for i, lay in enumerate(layers):
                lay.forward(cur, bufs[i % 2], want_info=False)
                cur = bufs[i % 2]
            return cur

        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            y_eager = run().clone()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                y_graph = run()
            g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y_graph.view(torch.int16), y_eager.view(torch.int16))
        for lay in layers:
            lay.close()
    finally:
        im.ep_comm_destroy(comm)
