"""Resident-layer FFN timing for kernel-knob sweeps (dev tool; bench.py is the
measurement of record).  Builds one resident layer (C2 by default; C5 with
--gate softmax --E 64 --k 2 --N 16384 --skew 1), runs it `--iters` times with
CUDA events, and prints one JSON line with the layer time, the fused FFN time
from the layer's own timeline, and a bitwise checksum of y, so runs under
different INFMOE_* environment knobs can be compared for speed and identity."""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2106_10715_b200 import device as dv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--gate", default="lsh")
ap.add_argument("--E", type=int, default=32)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--skew", type=float, default=0.0)
ap.add_argument("--c5", action="store_true",
                help="bench.py's C5 layer: SURVEY 8(d) Gaussian inputs at S5 = SEED + 500, "
                     "softmax top-2 over 64 experts, 16384 tokens, calibrated bias c = 0.6258")
a = ap.parse_args()
if a.c5:
    a.gate, a.E, a.k, a.N, a.skew = "softmax", 64, 2, 16384, 0.6258
d, f, E, N, k = 4096, 10240, a.E, a.N, a.k
dev = torch.device("cuda:0")
import paper_2106_10715_b200 as im  # noqa: E402
S = 20261018 + 500
hi = torch.empty((E, f, d), dtype=torch.bfloat16, pin_memory=True)
ho = torch.empty((E, d, f), dtype=torch.bfloat16, pin_memory=True)
seeds = [im.derive_seed(S, 1000 + 2 * e) for e in range(E)] + \
        [im.derive_seed(S, 1001 + 2 * e) for e in range(E)]
im.gaussian_fill_typed("bf16", seeds, [d ** -0.5] * E + [f ** -0.5] * E, f * d,
                       [hi[e].data_ptr() for e in range(E)] + [ho[e].data_ptr() for e in range(E)])
wi, wo = hi.to(dev), ho.to(dev)
del hi, ho
x = torch.from_numpy(im.gaussian_bf16(im.derive_seed(S, 0), N * d).view(np.int16)
                     .reshape(N, d)).view(torch.bfloat16).to(dev)
gw = np.ascontiguousarray((im.gaussian_stream(im.derive_seed(S, 1), d * E) * d ** -0.5)
                          .astype(np.float32).reshape(d, E).T)
bias = (-a.skew * np.log(np.arange(1, E + 1))).astype(np.float32)
layer = dv.MoELayer(d, f, E, k, wi, wo, gate=a.gate, gate_weight=gw, gate_bias=bias, lsh_seed=7,
                    lsh_bits=5, max_tokens=N)
y = torch.empty_like(x)
for _ in range(3):
    layer.forward(x, y, want_info=False)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
ts, ffn = [], []
for _ in range(a.iters):
    e0, e1 = ev(), ev()
    e0.record()
    layer.forward(x, y, want_info=False)
    e1.record()
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
    _, info = layer.forward(x, y, want_timeline=True)
    ffn.append((info["events"][0][4] - info["events"][0][3]) * 1e3)
flops = 4.0 * N * k * d * f
hbm = (int((info["counts"] > 0).sum()) * 2 * d * f + N * k * (2 * d + 2 * f)) * 2
t_bound = max(flops / 1643.6e12, hbm / 6549.1e9)
print(json.dumps({"env": {kk: v for kk, v in os.environ.items() if kk.startswith("INFMOE_")},
                  "layer_ms": float(np.median(ts)), "ffn_ms": float(np.median(ffn)),
                  "ffn_tflops": flops / (float(np.median(ffn)) * 1e-3) / 1e12,
                  "layer_over_t_bound": t_bound / (float(np.median(ts)) * 1e-3),
                  "max_rows": int(info["counts"].max()),
                  "y_sum": int(y.view(torch.int16).to(torch.int64).sum().item())}))
