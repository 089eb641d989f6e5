"""Quick per-stage timing of one resident MoE layer with CUDA events (dev tool;
bench.py is the measurement of record)."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--E", type=int, default=32)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--gate", default="lsh")
ap.add_argument("--k", type=int, default=1)
a = ap.parse_args()
d, f, E, N, k = 4096, 10240, a.E, a.N, a.k
dev = torch.device("cuda:0")
wi = torch.empty((E, f, d), dtype=torch.bfloat16, device=dev)
wo = torch.empty((E, d, f), dtype=torch.bfloat16, device=dev)
x = torch.empty((N, d), dtype=torch.bfloat16, device=dev)
dv.fill_uniform(wi, 1, 3 ** 0.5 / d ** 0.5)
dv.fill_uniform(wo, 2, 1.534 * 3 ** 0.5 / f ** 0.5)
dv.fill_uniform(x, 3, 3 ** 0.5)
proj = torch.from_numpy(im.gating_projection(7, 5, d)).to(dev)
gw = torch.randn(E, d, device=dev) / d ** 0.5
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def ev():
    return torch.cuda.Event(enable_timing=True)


def step_fused():
    """gate -> dispatch -> gather -> one-launch FFN with the top-1 combine fused"""
    e = [ev() for _ in range(5)]
    torch.cuda._sleep(20_000_000)
    e[0].record()
    if a.gate == "lsh":
        _, idx, w, cnt = dv.gate_lsh(x, proj, E)
    else:
        idx, w, cnt = dv.gate_softmax_topk(x, gw, k)
    off, perm, inv = dv.dispatch(idx, E)
    e[1].record()
    xp = dv.gather_rows(x, perm, k)
    e[2].record()
    if k == 1:
        dv.expert_ffn_fused(xp, off, wi, wo, perm=perm, topk_w=w.reshape(-1), n_tokens=N)
        e[3].record()
        e[4].record()
    else:
        _, yp = dv.expert_ffn_fused(xp, off, wi, wo)
        e[3].record()
        dv.combine(yp, inv, w, N, k)
        e[4].record()
    torch.cuda.synchronize()
    return [e[i].elapsed_time(e[i + 1]) for i in range(4)]


def step():
    e = [ev() for _ in range(7)]
    torch.cuda._sleep(20_000_000)  # ~10 ms: the host queues every launch before e[0] fires
    e[0].record()
    if a.gate == "lsh":
        _, idx, w, cnt = dv.gate_lsh(x, proj, E)
    else:
        idx, w, cnt = dv.gate_softmax_topk(x, gw, k)
    e[1].record()
    off, perm, inv = dv.dispatch(idx, E)
    e[2].record()
    xp = dv.gather_rows(x, perm, k)
    e[3].record()
    h, yp = dv.expert_ffn(xp, off, wi, wo)
    e[4].record()
    y = dv.combine(yp, inv, w, N, k)
    e[5].record()
    torch.cuda.synchronize()
    return [e[i].elapsed_time(e[i + 1]) for i in range(5)], cnt


names = ["gate", "dispatch", "gather", "expert_ffn", "combine"]
acc = [0.0] * 5
for i in range(a.iters + 3):
    flush.zero_()
    t, cnt = step()
    if i >= 3:
        acc = [p + q for p, q in zip(acc, t)]
acc = [v / a.iters for v in acc]
wbytes = E * 2 * d * f * 2
act = N * k * (2 * d + 2 * f) * 2
out = {n: round(v * 1e3, 1) for n, v in zip(names, acc)}
out["total_us"] = round(sum(acc) * 1e3, 1)
out["ffn_GBps"] = round((wbytes + act) / (acc[3] * 1e-3) / 1e9, 1)
out["counts_minmax"] = [int(cnt.min()), int(cnt.max())]
fz = [0.0] * 4
for i in range(a.iters + 3):
    flush.zero_()
    t = step_fused()
    if i >= 3:
        fz = [p + q for p, q in zip(fz, t)]
fz = [v / a.iters for v in fz]
out["fused"] = {"route_us": round(fz[0] * 1e3, 1), "gather_us": round(fz[1] * 1e3, 1),
                "ffn_fused_us": round(fz[2] * 1e3, 1), "combine_us": round(fz[3] * 1e3, 1),
                "total_us": round(sum(fz) * 1e3, 1),
                "ffn_GBps": round((wbytes + act) / (fz[2] * 1e-3) / 1e9, 1)}
print(json.dumps(out))
