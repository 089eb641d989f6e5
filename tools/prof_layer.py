"""Profiling driver: one resident C2 (or, with --gate softmax --E 64 --k 2 --N 16384
--skew 1, C5) layer (d4096 f10240 E32 top-1 LSH, 4096
tokens, bf16) run `--iters` times; used under ncu (never timed for results)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--gate", default="lsh")
ap.add_argument("--E", type=int, default=32)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--skew", type=float, default=0.0, help="softmax logit bias -skew*ln(e+1) (C5: 1)")
a = ap.parse_args()
d, f, E, N = 4096, 10240, a.E, a.N
dev = torch.device("cuda:0")
wi = torch.empty((E, f, d), dtype=torch.bfloat16, device=dev)
wo = torch.empty((E, d, f), dtype=torch.bfloat16, device=dev)
x = torch.empty((N, d), dtype=torch.bfloat16, device=dev)
dv.fill_uniform(wi, 1, 3 ** 0.5 / d ** 0.5)
dv.fill_uniform(wo, 2, 1.534 * 3 ** 0.5 / f ** 0.5)
dv.fill_uniform(x, 3, 3 ** 0.5)
gw = torch.randn(E, d).numpy() / d ** 0.5
bias = -a.skew * torch.log(torch.arange(1, E + 1, dtype=torch.float32)).numpy()
layer = dv.MoELayer(d, f, E, a.k, wi, wo, gate=a.gate, gate_weight=gw, gate_bias=bias, lsh_seed=7,
                    lsh_bits=5, max_tokens=N)
y = torch.empty_like(x)
for _ in range(a.iters):
    layer.forward(x, y, want_info=False)
torch.cuda.synchronize()
print("ok")
