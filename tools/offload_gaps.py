"""Dev tool: where does the host link idle in the offloaded executor?

Runs a short offloaded LSH stack (bench.py's C3 shapes) with timelines and
reports, per layer: time to the first load, the sum of load durations, the
gaps between consecutive loads, and the tail after the last load.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2106_10715_b200 as im  # noqa: E402
from paper_2106_10715_b200 import device as dv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--codec", default="raw", choices=["raw", "exp4", "exph"])
    a = ap.parse_args()
    d, f, E, N = 4096, 10240, 32, 4096
    bf = torch.bfloat16
    dev = torch.device("cuda:0")
    hi = torch.empty((E, f, d), dtype=bf, pin_memory=True)
    ho = torch.empty((E, d, f), dtype=bf, pin_memory=True)
    bench.fill_expert_weights(im, bench.SEED, 0, E, d, f, hi, ho)  # SURVEY 8(d) weights
    x = torch.from_numpy(im.gaussian_bf16(im.derive_seed(bench.SEED, 0), N * d).view(np.int16)
                         .reshape(N, d)).view(bf).to(dev)
    pool = dv.SlotPool(4, d, f)
    layers = [dv.MoELayer(d, f, E, 1, hi, ho, gate="lsh", lsh_seed=bench.lsh_seed(im, l),
                          lsh_bits=5, offloaded=True, K=4, max_tokens=N, h2d_codec=a.codec,
                          slot_pool=pool)
              for l in range(a.layers)]
    bufs = [torch.empty_like(x) for _ in range(2)]
    for rep in range(2):
        cur = x
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        infos = []
        for l, layer in enumerate(layers):
            _, info = layer.forward(cur, bufs[l % 2], want_timeline=True, time_origin=t0)
            infos.append(info)
            cur = bufs[l % 2]
        t1 = torch.cuda.Event(enable_timing=True)
        t1.record()
        torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    nbytes = layers[0].packed_bytes() / E  # bytes per expert load over the link
    prev_end = 0.0
    for l, info in enumerate(infos):  # times on one axis: seconds from t0
        loads = sorted([(s0, s1) for st, _, _, s0, s1 in info["events"] if st == 0])
        comps = sorted([(s0, s1) for st, _, _, s0, s1 in info["events"] if st == 1])
        dur = [b - a for a, b in loads]
        gaps = [loads[i + 1][0] - loads[i][1] for i in range(len(loads) - 1)]
        end = max(c[1] for c in comps)
        print(f"layer {l}: head (prev layer end -> first load) {(loads[0][0] - prev_end) * 1e3:.3f} ms, "
              f"loads {sum(dur) * 1e3:.2f} ms (mean {np.mean(dur) * 1e3:.3f} ms = "
              f"{nbytes / np.mean(dur) / 1e9:.2f} GB/s), gaps sum {sum(gaps) * 1e3:.3f} ms max "
              f"{max(gaps) * 1e6:.1f} us, tail (last load end -> last compute end) "
              f"{(end - loads[-1][1]) * 1e3:.3f} ms [last compute {(comps[-1][1] - comps[-1][0]) * 1e3:.3f} ms "
              f"started {(comps[-1][0] - loads[-1][1]) * 1e6:.1f} us after its load]")
        prev_end = end
    print(f"stack {total:.2f} ms, ideal at per-load rate {a.layers * E * np.mean(dur) * 1e3:.2f} ms")
    for layer in layers:
        layer.close()


if __name__ == "__main__":
    main()
