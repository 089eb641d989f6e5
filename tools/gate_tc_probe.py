"""Dev probe: the C5 softmax gate (N=16384, d=4096, E=64, top-2, calibrated
Zipf bias) through the C-ABI, tensor-core path then CUDA-core path
(INFMOE_GATE_TC=0); run under ncu for per-kernel times."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

N, d, E, k = 16384, 4096, 64, 2
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 29
xb = im.gaussian_bf16(im.derive_seed(seed, 0), N * d)
wg = np.ascontiguousarray((im.gaussian_stream(im.derive_seed(seed, 1), d * E) /
                           np.sqrt(d)).astype(np.float32).reshape(d, E).T)
bias = (-0.6258 * np.log(np.arange(1, E + 1))).astype(np.float32)
x = torch.from_numpy(xb.view(np.int16).reshape(N, d)).cuda().view(torch.bfloat16)
g, b = torch.from_numpy(wg).cuda(), torch.from_numpy(bias).cuda()
ws = dv.GateWorkspace(g, N, k)  # as a layer holds it
out = dv.gate_softmax_topk(x, g, k, b, debug=True)
print("gate stats", out[4], "exact chains per fallback token",
      out[4]["candidates"] / max(out[4]["fallback"], 1))
for _ in range(3):
    dv.gate_softmax_topk(x, g, k, b, workspace=ws)
os.environ["INFMOE_GATE_TC"] = "0"
for _ in range(2):
    dv.gate_softmax_topk(x, g, k, b)
torch.cuda.synchronize()
