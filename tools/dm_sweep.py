"""Data-movement kernels of the path at C5 sizes (16384 tokens x 4096, E=64,
top-2): softmax gate, dispatch, gather, combine — median of `--iters` launches,
each after a 256 MB L2 flush, CUDA events (dev tool; bench.py's
`c5.data_movement` is the measurement of record).  Prints a checksum of every
output so kernel variants can be compared for identity."""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2106_10715_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=9)
ap.add_argument("--N", type=int, default=16384)
ap.add_argument("--E", type=int, default=64)
ap.add_argument("--k", type=int, default=2)
a = ap.parse_args()
N, d, E, k = a.N, 4096, a.E, a.k
dev = torch.device("cuda:0")
x = torch.empty((N, d), dtype=torch.bfloat16, device=dev)
dv.fill_uniform(x, 3, 3 ** 0.5)
gw = torch.from_numpy((np.random.default_rng(5).standard_normal((E, d)) / d ** 0.5)
                      .astype(np.float32)).to(dev)
bias = torch.from_numpy((-np.log(np.arange(1, E + 1))).astype(np.float32)).to(dev)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ev = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn):
    ts = []
    for _ in range(a.iters):
        flush_buf.zero_()
        e0, e1 = ev(), ev()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


idx, w, cnt = dv.gate_softmax_topk(x, gw, k, bias=bias)
off, perm, inv = dv.dispatch(idx, E)
xp = dv.gather_rows(x, perm, k)
y = dv.combine(xp, inv, w, N, k)
torch.cuda.synchronize()
t_gate = timed(lambda: dv.gate_softmax_topk(x, gw, k, bias=bias))
t_disp = timed(lambda: dv.dispatch(idx, E))
t_gath = timed(lambda: dv.gather_rows(x, perm, k))
t_gtok = timed(lambda: dv.gather_rows_by_token(x, inv, k))
t_comb = timed(lambda: dv.combine(xp, inv, w, N, k))
gath_b = N * d * 2 + N * k * d * 2 + N * k * 4
comb_b = N * k * d * 2 + N * d * 2 + N * k * 8
cs = lambda t: int(t.contiguous().view(torch.int32).to(torch.int64).sum().item()) if t.element_size() == 4 \
    else int(t.view(torch.int16).to(torch.int64).sum().item())
print(json.dumps({"gate_us": t_gate * 1e6, "dispatch_us": t_disp * 1e6,
                  "gather_us": t_gath * 1e6, "gather_gbs": gath_b / t_gath / 1e9,
                  "gather_by_token_us": t_gtok * 1e6, "gather_by_token_gbs": gath_b / t_gtok / 1e9,
                  "combine_us": t_comb * 1e6, "combine_gbs": comb_b / t_comb / 1e9,
                  "checksums": [cs(idx), cs(w), cs(perm), cs(xp), cs(y)]}))
