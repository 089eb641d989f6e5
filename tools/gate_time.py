"""Softmax gate timing at C5 size (16384 x 4096, E = 64, top-2; Gaussian inputs,
calibrated bias), CUDA events over 10 back-to-back launches after an L2 flush,
plus a checksum of the routing so kernel variants can be
compared for speed and identity (dev tool)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

N, d, E, k = 16384, 4096, 64, 2
dev = torch.device("cuda:0")
S = 20261018 + 500
x = torch.from_numpy(im.gaussian_bf16(im.derive_seed(S, 0), N * d).view(np.int16)
                     .reshape(N, d)).view(torch.bfloat16).to(dev)
gw = torch.from_numpy(np.ascontiguousarray((im.gaussian_stream(im.derive_seed(S, 1), d * E) *
                                            d ** -0.5).astype(np.float32).reshape(d, E).T)).to(dev)
bias = torch.from_numpy((-0.6258 * np.log(np.arange(1, E + 1))).astype(np.float32)).to(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for E_ in (64, 32):
    g = gw[:E_].contiguous()
    b = bias[:E_].contiguous()
    for _ in range(3):
        idx, w, cnt = dv.gate_softmax_topk(x, g, k, bias=b)
    ts = []
    for _ in range(5):
        flush.zero_()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            dv.gate_softmax_topk(x, g, k, bias=b)
        z.record()
        z.synchronize()
        ts.append(a.elapsed_time(z) / 10 * 1e3)
    print(f"E={E_}: {np.median(ts):.1f} us  idx_sum={int(idx.long().sum())} "
          f"w_sum={float(w.double().sum()):.6f} counts_max={int(cnt.max())}")
