"""The fused expert FFN on one GPU for E_local = 4 / 8 / 16 / 32 experts of ~128
rows each (the per-rank shape of the C4 expert-parallel stack at P = 8 / 4 / 2
/ 1), CPM-2 expert size, bf16: per-launch time (CUDA events, median of 20
back-to-back launches after an L2 flush) and algorithmic HBM GB/s (weights
once + x_perm + H write/read + y) against MEASURED_PEAKS.json (dev tool)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

d, f, rows = 4096, 10240, 128
dev = torch.device("cuda:0")
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6549.1
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
g = torch.Generator(device="cpu").manual_seed(1)
for E in [int(v) for v in sys.argv[1:]] or (4, 8, 16, 32):
    counts = [rows + (e % 3) * 7 - 7 for e in range(E)]
    R = sum(counts)
    offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=dev)
    x = torch.randn(R, d, generator=g).to(torch.bfloat16).to(dev)
    wi = (torch.randn(E, f, d, generator=g) / d ** 0.5).to(torch.bfloat16).to(dev)
    wo = (torch.randn(E, d, f, generator=g) / f ** 0.5).to(torch.bfloat16).to(dev)
    kw = {}
    for _ in range(3):
        dv.expert_ffn_fused(x, offs, wi, wo, **kw)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dv.expert_ffn_fused(x, offs, wi, wo, **kw)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = float(np.median(ts))
    alg = E * 2 * d * f * 2 + R * (2 * d + 2 * f) * 2
    print(json.dumps({"experts": E, "rows": R, "us": t * 1e6, "alg_gbs": alg / t / 1e9,
                      "frac_of_hbm": alg / t / 1e9 / peak}))
    del x, wi, wo
    torch.cuda.empty_cache()
