"""Profiling driver for the data-movement kernels of the path at C5 size
(16384 tokens x d 4096, top-2 over E = 64, bf16; SURVEY 8(d) Gaussian inputs,
logit bias -c ln(e+1) with bench.py's calibrated c) plus the LSH gate at C2:
softmax gate, dispatch (counting sort), gather_rows_by_token, combine, and the
LSH gate, each launched --iters times.  Target for `ncu --set full` (never timed
for results; bench.py's c5.data_movement is the CUDA-event measurement)."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--c", type=float, default=0.6258)
a = ap.parse_args()
N, d, E, k = 16384, 4096, 64, 2
dev = torch.device("cuda:0")
S = 20261018 + 500
xb = im.gaussian_bf16(im.derive_seed(S, 0), N * d)
x = torch.from_numpy(xb.view(np.int16).reshape(N, d)).view(torch.bfloat16).to(dev)
gw = torch.from_numpy(np.ascontiguousarray(
    (im.gaussian_stream(im.derive_seed(S, 1), d * E) * d ** -0.5).astype(np.float32)
    .reshape(d, E).T)).to(dev)
bias = torch.from_numpy((-a.c * np.log(np.arange(1, E + 1))).astype(np.float32)).to(dev)
proj = torch.from_numpy(im.gating_projection(im.derive_seed(20261018, 2), 5, d)).to(dev)
x2 = x[:4096].contiguous()
for _ in range(a.iters):
    idx, w, cnt = dv.gate_softmax_topk(x, gw, k, bias=bias)
    offs, perm, inv = dv.dispatch(idx, E)
    xp = dv.gather_rows_by_token(x, inv, k)
    y = dv.combine(xp, inv, w, N, k)
    dv.gate_lsh(x2, proj, 32)
torch.cuda.synchronize()
print("ok", cnt.max().item())
