"""Dev probe: HBM copy bandwidth burst vs sustained on this box (the
denominator question for a power-capped kernel).  torch copy_ of 1 GiB bf16
(read + write bytes), best single copy vs ~N seconds back to back, with
nvidia-smi clocks sampled during the sustained run."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    n = 1 << 30
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1.0)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0, e1 = ev(), ev()
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    burst = 2 * n * 2 / (best * 1e-3) / 1e9
    reps = int(float(sys.argv[1]) * 1e3 / best) if len(sys.argv) > 1 else 12000 // int(best + 1)
    e0, e1 = ev(), ev()
    with bench.ClockSampler(0) as ck:
        e0.record()
        for _ in range(reps):
            b.copy_(a)
        e1.record()
        e1.synchronize()
    sus = 2 * n * 2 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(f"burst {burst:.1f} GB/s, sustained {sus:.1f} GB/s over {e0.elapsed_time(e1) / 1e3:.1f} s, "
          f"clocks {ck.summary()}, power {[r[3] for r in ck.rows][-5:]}")


if __name__ == "__main__":
    main()
