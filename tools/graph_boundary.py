"""Dev probe: cost of the kernel boundaries around the fused FFN inside a CUDA
graph.  Same inputs, three graphs of 24 repetitions: [FFN], [gather, FFN],
[gate, dispatch, gather, FFN]; prints ms per repetition for each."""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    d, f, N, L = 4096, 10240, 128 * E, 24
    dev = torch.device("cuda:0")
    bf = torch.bfloat16
    ws = []
    for s in range(4):
        wi = torch.empty((E, f, d), dtype=bf, device=dev)
        wo = torch.empty((E, d, f), dtype=bf, device=dev)
        for e in range(E):
            dv.fill_uniform(wi[e], im.derive_seed(bench.SEED, 10_000 * (s + 1) + 2 * e), bench.SQRT3 / d ** 0.5)
            dv.fill_uniform(wo[e], im.derive_seed(bench.SEED, 10_000 * (s + 1) + 2 * e + 1),
                            bench.GELU_GAIN * bench.SQRT3 / f ** 0.5)
        ws.append((wi, wo))
    x = torch.empty((N, d), dtype=bf, device=dev)
    dv.fill_uniform(x, im.derive_seed(bench.SEED, 0), math.sqrt(3.0))
    proj = torch.from_numpy(np.ascontiguousarray(im.gating_projection(im.derive_seed(bench.SEED, 100), 5, d))).to(dev)
    _, idx, w, _ = dv.gate_lsh(x, proj, E)  # E <= 32 with 5 bits
    off, perm, _ = dv.dispatch(idx, E)
    xp = dv.gather_rows(x, perm, 1)
    torch.cuda.synchronize()

    def ffn(l):
        dv.expert_ffn_fused(xp, off, *ws[l % 4], perm=perm, topk_w=w.reshape(-1), n_tokens=N)

    def gather(l):
        dv.gather_rows(x, perm, 1)

    def route(l):
        _, i2, _, _ = dv.gate_lsh(x, proj, E)
        dv.dispatch(i2, E)

    variants = {"ffn": [ffn], "gather+ffn": [gather, ffn], "gate+dispatch+gather+ffn": [route, gather, ffn]}
    for name, parts in variants.items():
        for _ in range(2):
            for l in range(L):
                for p in parts:
                    p(l)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for l in range(L):
                for p in parts:
                    p(l)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:28s} {e0.elapsed_time(e1) / (3 * L) * 1e3:8.1f} us per repetition")
        del g


if __name__ == "__main__":
    main()
