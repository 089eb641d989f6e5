"""Dev tool: per-layer routing skew and fused-FFN time of bench.py's resident stack.

Builds the same 24-layer LSH stack as bench.py (4 aliased weight sets), runs
one timeline pass and prints, per layer, the largest expert's rows, the number
of non-empty experts and the fused expert-FFN kernel time.
"""
import argparse
import math

import numpy as np
import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (constants only)
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402

SEED = bench.SEED


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--sets", type=int, default=4)
    ap.add_argument("--extra-gb", type=float, default=0.0, help="extra idle device allocation")
    ap.add_argument("--burn", type=int, default=0, help="untimed stack passes first")
    ap.add_argument("--offload-passes", type=int, default=0, help="offloaded stack passes first")
    ap.add_argument("--pinned-gb", type=float, default=0.0, help="pinned host pool, streamed once")
    ap.add_argument("--sleep", type=float, default=0.0, help="idle seconds first")
    ap.add_argument("--smi", type=float, default=0.0, help="seconds of nvidia-smi sampling first")
    a = ap.parse_args()
    d, f, E, N = 4096, 10240, 32, a.tokens
    bf = torch.bfloat16
    dev = torch.device("cuda:0")
    ws = []
    for s in range(a.sets):
        wi = torch.empty((E, f, d), dtype=bf, device=dev)
        wo = torch.empty((E, d, f), dtype=bf, device=dev)
        for e in range(E):
            dv.fill_uniform(wi[e], im.derive_seed(SEED, 10_000 * (s + 1) + 2 * e),
                            bench.SQRT3 / d ** 0.5)
            dv.fill_uniform(wo[e], im.derive_seed(SEED, 10_000 * (s + 1) + 2 * e + 1),
                            bench.GELU_GAIN * bench.SQRT3 / f ** 0.5)
        ws.append((wi, wo))
    x = torch.empty((N, d), dtype=bf, device=dev)
    dv.fill_uniform(x, im.derive_seed(SEED, 0), math.sqrt(3.0))
    layers = [dv.MoELayer(d, f, E, 1, *ws[l % a.sets], gate="lsh",
                          lsh_seed=im.derive_seed(SEED, 100 + l), lsh_bits=5,
                          offloaded=False, max_tokens=N) for l in range(a.layers)]
    bufs = [torch.empty_like(x) for _ in range(2)]
    extra = torch.empty(int(a.extra_gb * (1 << 30)), dtype=torch.uint8, device=dev) if a.extra_gb else None
    for _ in range(a.burn):
        cur = x
        for l, layer in enumerate(layers):
            layer.forward(cur, bufs[l % 2], want_info=False)
            cur = bufs[l % 2]
    if a.offload_passes:
        hs = []
        for wi, wo in ws[:1]:
            hi = torch.empty(wi.shape, dtype=bf, pin_memory=True)
            ho = torch.empty(wo.shape, dtype=bf, pin_memory=True)
            hi.copy_(wi)
            ho.copy_(wo)
            hs.append((hi, ho))
        off = [dv.MoELayer(d, f, E, 1, *hs[0], gate="lsh", lsh_seed=im.derive_seed(SEED, 100 + l),
                           lsh_bits=5, offloaded=True, K=4, max_tokens=N) for l in range(4)]
        for _ in range(a.offload_passes):
            cur = x
            for l, layer in enumerate(off):
                layer.forward(cur, bufs[l % 2], want_info=False)
                cur = bufs[l % 2]
        torch.cuda.synchronize()
        print("offload passes done")
    if a.pinned_gb:
        pool = torch.empty(int(a.pinned_gb * (1 << 30)), dtype=torch.uint8, pin_memory=True)
        pool.fill_(1)
        chunk = 1 << 28
        dst = torch.empty(chunk, dtype=torch.uint8, device=dev)
        for o in range(0, pool.numel(), chunk):
            n = min(chunk, pool.numel() - o)
            dst[:n].copy_(pool[o:o + n], non_blocking=True)
        torch.cuda.synchronize()
        print("pinned pool streamed")
    if a.sleep:
        import time
        time.sleep(a.sleep)
    if a.smi:
        import time
        with bench.ClockSampler(0):
            time.sleep(a.smi)
    torch.cuda.synchronize()
    tot = []
    for rep in range(2):
        cur = x
        for l, layer in enumerate(layers):
            y = bufs[l % 2]
            _, info = layer.forward(cur, y, want_timeline=True)
            cur = y
            if rep == 1:
                rows = info["local_rows"]
                ev = info["events"][0]
                us = (ev[4] - ev[3]) * 1e6
                tot.append(us)
                by = int((rows > 0).sum()) * 2 * d * f * 2 + int(rows.sum()) * (2 * d + 2 * f) * 2
                print(f"layer {l:2d}: max_rows {int(rows.max()):5d} nonempty {int((rows > 0).sum()):2d} "
                      f"ffn {us:8.1f} us  {by / us / 1e3:7.1f} GB/s  std(x) {cur.float().std().item():.3f}")
    print(f"mean ffn {sum(tot) / len(tot):.1f} us")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(0) as ck:
        e0.record()
        for _ in range(20):
            cur = x
            for l, layer in enumerate(layers):
                layer.forward(cur, bufs[l % 2], want_info=False)
                cur = bufs[l % 2]
        e1.record()
        torch.cuda.synchronize()
    print(f"stack pass {e0.elapsed_time(e1) / 20:.3f} ms ({e0.elapsed_time(e1) / 20 / len(layers) * 1e3:.1f} us/layer)")
    # the same stack as one CUDA graph (bench.py's resident path)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = x
        for l, layer in enumerate(layers):
            layer.forward(cur, bufs[l % 2], want_info=False)
            cur = bufs[l % 2]
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph pass {e0.elapsed_time(e1) / 20:.3f} ms ({e0.elapsed_time(e1) / 20 / len(layers) * 1e3:.1f} us/layer)")
    print("clocks", ck.summary(), "power", [r[3] for r in ck.rows][:12])
    del extra
    for layer in layers:
        layer.close()


if __name__ == "__main__":
    main()
