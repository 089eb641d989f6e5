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
# SURVEY 8(d) inputs, as bench.py: GaussianStream weights x d^-1/2 / f^-1/2,
# gaussian_tokens x, all rounded to bf16 on the host
S = 20261018
wi = torch.empty((E, f, d), dtype=torch.bfloat16, pin_memory=True)
wo = torch.empty((E, d, f), dtype=torch.bfloat16, pin_memory=True)
x = torch.empty((N, d), dtype=torch.bfloat16, pin_memory=True)
im.gaussian_fill_typed("bf16", [im.derive_seed(S, 1000 + 2 * e) for e in range(E)] +
                       [im.derive_seed(S, 1001 + 2 * e) for e in range(E)],
                       [d ** -0.5] * E + [f ** -0.5] * E, f * d,
                       [wi[e].data_ptr() for e in range(E)] + [wo[e].data_ptr() for e in range(E)])
im.gaussian_fill_typed("bf16", [im.derive_seed(S, 0)], [1.0], N * d, [x.data_ptr()])
wi, wo, x = wi.to(dev), wo.to(dev), x.to(dev)
gw = torch.randn(E, d).numpy() / d ** 0.5
bias = -a.skew * torch.log(torch.arange(1, E + 1, dtype=torch.float32)).numpy()
layer = dv.MoELayer(d, f, E, a.k, wi, wo, gate=a.gate, gate_weight=gw, gate_bias=bias, lsh_seed=7,
                    lsh_bits=5, max_tokens=N)
y = torch.empty_like(x)
for _ in range(a.iters):
    layer.forward(x, y, want_info=False)
torch.cuda.synchronize()
print("ok")
