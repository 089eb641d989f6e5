"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck)
over the persistent fused expert FFN (pair and one-SM kernels, with the
dynamic tile claim and the cross-CTA H-ready counters), the LSH / softmax
gates, dispatch, gather, combine and the exph decoder, plus one offloaded
layer forward.  Usage:
  compute-sanitizer --tool racecheck python tools/sanitize_ffn.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_10715_b200 import device as dv  # noqa: E402

cuda = torch.device("cuda:0")
g = torch.Generator(device="cpu").manual_seed(3)
E, d, f = 4, 256, 512
counts = [40, 0, 130, 17]
R = sum(counts)
offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=cuda)
x = torch.randn(R, d, generator=g).to(torch.bfloat16).to(cuda)
wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(cuda)
wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(cuda)
h, y = dv.expert_ffn_fused(x, offs, wi, wo)
torch.cuda.synchronize()

N = 96
xt = torch.randn(N, d, generator=g).to(torch.bfloat16).to(cuda)
wg = (torch.randn(E, d, generator=g) / d ** 0.5).to(cuda)
idx, w, cnt = dv.gate_softmax_topk(xt, wg, 2)
o, perm, inv = dv.dispatch(idx, E)
xp = dv.gather_rows_by_token(xt, inv, 2)
yc = dv.combine(xp, inv, w, N, 2)
torch.cuda.synchronize()

if os.environ.get("SAN_LAYER", "1") == "1":
    lay = dv.MoELayer(d, f, E, 1, wi.cpu().pin_memory(), wo.cpu().pin_memory(), gate="lsh",
                      lsh_seed=3, lsh_bits=2, max_tokens=N, offloaded=True, K=1,
                      h2d_codec="exph")
    yl, info = lay.forward(xt)
    torch.cuda.synchronize()
    lay.close()
print("sanitize driver ok", os.environ.get("INFMOE_FFN_PAIR", "1"))
