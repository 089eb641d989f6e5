"""Expert parallelism across 2 processes on CPU (gloo): the product's EP plan
(libinfmoe.so infmoe_ep_plan, host code) drives a real two-rank all-to-allv of
routed token rows; each rank runs only its experts (CPU oracle FFN) and the
result must equal the single-process layer bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N, D, F, E, K_TOP = 96, 64, 96, 8, 2


def _problem():
    from oracle_lib import bf16_bits_to_f32, fill_bf16
    x = bf16_bits_to_f32(fill_bf16(1, N * D, 1.7320508)).reshape(N, D)
    wi = bf16_bits_to_f32(fill_bf16(2, E * F * D, 1.7320508 / D ** 0.5)).reshape(E, F, D)
    wo = bf16_bits_to_f32(fill_bf16(3, E * D * F, 1.534 * 1.7320508 / F ** 0.5)).reshape(E, D, F)
    wg = (np.random.default_rng(4).standard_normal((E, D)) / D ** 0.5).astype(np.float32)
    return x, wi, wo, wg


def _layer_cpu(x, wi, wo, wg, experts_here=None, rows_in=None):
    """oracle chain; returns (y, idx, w, perm, inv, offsets, y_perm)"""
    from oracle_lib import O, ptr
    n = x.shape[0]
    idx = np.zeros((n, K_TOP), np.int32)
    w = np.zeros((n, K_TOP), np.float32)
    cnt = np.zeros(E, np.int32)
    O.or_gate_softmax(ptr(np.ascontiguousarray(x)), n, D, ptr(wg), None, E, K_TOP, ptr(idx),
                      ptr(w), ptr(cnt))
    off = np.zeros(E + 1, np.int32)
    perm = np.zeros(n * K_TOP, np.int32)
    inv = np.zeros(n * K_TOP, np.int32)
    O.or_dispatch(ptr(idx), n, K_TOP, E, ptr(off), ptr(perm), ptr(inv))
    return idx, w, cnt, off, perm, inv


def _ffn(rows, wi_e, wo_e):
    from oracle_lib import O, ptr
    y = np.zeros((rows.shape[0], D), np.float32)
    if rows.shape[0]:
        O.or_expert_ffn(ptr(np.ascontiguousarray(rows)), rows.shape[0], D, F,
                        ptr(np.ascontiguousarray(wi_e)), ptr(np.ascontiguousarray(wo_e)), 1,
                        ptr(y))
    return y


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2106_10715_b200 as im
        from oracle_lib import O, ptr
        x, wi, wo, wg = _problem()
        El = E // world
        shard = x[rank * N // world:(rank + 1) * N // world]
        n = shard.shape[0]
        idx, w, cnt, off, perm, inv = _layer_cpu(shard, wi, wo, wg)
        xp = np.ascontiguousarray(shard[perm // K_TOP])
        # count exchange: rows for each peer's experts
        send_c = torch.from_numpy(cnt.copy())
        recv_c = torch.empty(world * El, dtype=torch.int32)
        dist.all_to_all_single(recv_c, send_c)
        plan = im.ep_plan(world, rank, E, cnt, recv_c.numpy())
        # token all-to-allv
        recv = torch.empty((plan.n_recv, D), dtype=torch.float32)
        dist.all_to_all_single(recv, torch.from_numpy(xp), plan.recv_rows.tolist(),
                               plan.send_rows.tolist())
        loc = recv.numpy()[plan.local_index]
        ly = np.zeros_like(loc)
        for e in range(El):
            a, b = plan.local_offsets[e], plan.local_offsets[e + 1]
            ge = rank * El + e
            ly[a:b] = _ffn(loc[a:b], wi[ge], wo[ge])
        back = np.zeros_like(loc)
        back[plan.local_index] = ly
        yp = torch.empty((n * K_TOP, D), dtype=torch.float32)
        dist.all_to_all_single(yp, torch.from_numpy(back), plan.send_rows.tolist(),
                               plan.recv_rows.tolist())
        y = np.zeros((n, D), np.float32)
        O.or_combine(ptr(np.ascontiguousarray(yp.numpy())), ptr(inv), ptr(w), n, K_TOP, D, ptr(y))
        # single-process reference for the same shard
        ref_yp = np.zeros((n * K_TOP, D), np.float32)
        for e in range(E):
            a, b = off[e], off[e + 1]
            ref_yp[a:b] = _ffn(xp[a:b], wi[e], wo[e])
        ref = np.zeros((n, D), np.float32)
        O.or_combine(ptr(ref_yp), ptr(inv), ptr(w), n, K_TOP, D, ptr(ref))
        q.put((rank, bool(np.array_equal(y, ref)), int(plan.n_recv)))
    except Exception as ex:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(ex), -1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_ep_two_ranks_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(ok is True for _, ok, _ in res), res
    assert sum(n for _, _, n in res) == N * K_TOP  # every routed row served exactly once


def test_ep_plan_properties():
    import paper_2106_10715_b200 as im
    rng = np.random.default_rng(0)
    for P in (1, 2, 4, 8):
        E2 = 8 * P
        El = E2 // P
        allc = rng.integers(0, 50, (P, E2)).astype(np.int32)  # allc[src][global expert]
        for r in range(P):
            recv = allc[:, r * El:(r + 1) * El].reshape(-1)
            plan = im.ep_plan(P, r, E2, allc[r], recv)
            assert plan.send_rows.tolist() == [int(allc[r, q * El:(q + 1) * El].sum())
                                               for q in range(P)]
            assert plan.recv_rows.tolist() == [int(allc[s, r * El:(r + 1) * El].sum())
                                               for s in range(P)]
            assert plan.n_recv == int(recv.sum())
            assert sorted(plan.local_index.tolist()) == list(range(plan.n_recv))
            assert np.diff(plan.local_offsets).tolist() == allc[:, r * El:(r + 1) * El].sum(0).tolist()
    with pytest.raises(ValueError):
        im.ep_plan(3, 0, 8, np.zeros(8), np.zeros(8))  # E not a multiple of P
