"""Dev probe: the host link for expert-sized copies (112 MB, an exph pack pair):
24 back-to-back copies on one stream (the executor's load lane) vs alternating
two streams, vs one 1 GiB copy; CUDA events, best of 3 (dev tool)."""
import torch

dev = torch.device("cuda:0")
sz, n = 112 << 20, 24
h = torch.empty(n * sz, dtype=torch.uint8, pin_memory=True)
d = [torch.empty(sz, dtype=torch.uint8, device=dev) for _ in range(5)]
big = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(mode):
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        s2.wait_event(a)
        if mode == "big":
            with torch.cuda.stream(s1):
                big.copy_(h[: 1 << 30], non_blocking=True)
        else:
            for i in range(n):
                s = s1 if (mode == "one" or i % 2 == 0) else s2
                with torch.cuda.stream(s):
                    d[i % 5].copy_(h[i * sz:(i + 1) * sz], non_blocking=True)
        e2 = torch.cuda.Event()
        e2.record(s2)
        s1.wait_event(e2)
        b.record(s1)
        b.synchronize()
        nbytes = (1 << 30) if mode == "big" else n * sz
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


for m in ("big", "one", "two", "one", "two"):
    print(m, f"{run(m):.2f} GB/s")

# the same copies while another stream keeps HBM busy for the whole
# measurement (device-to-device copies of 1 GiB, like the decoder / FFN
# traffic beside the load lane)
src = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
dst = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
s3 = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(s3):
    for _ in range(700):  # ~230 ms of HBM traffic, longer than the 3 x 48 ms measured
        dst.copy_(src, non_blocking=True)
print("one, HBM busy beside it", f"{run('one'):.2f} GB/s")
torch.cuda.synchronize()


# copies that start at 16-byte (not page) aligned offsets with ragged sizes,
# like the packs (per-expert offsets in one pinned buffer, 16-aligned)
def run_ragged(align=16):
    best = 0.0
    sizes = [sz - 4096 * 7 - 16 * (i * 37 % 251) for i in range(n)]
    offs = [0]
    for z in sizes[:-1]:
        offs.append((offs[-1] + z + align - 1) // align * align)
    for _ in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s1)
        with torch.cuda.stream(s1):
            for i in range(n):
                d[i % 5][:sizes[i]].copy_(h[offs[i]:offs[i] + sizes[i]], non_blocking=True)
        b.record(s1)
        b.synchronize()
        best = max(best, sum(sizes) / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


for al in (16, 256, 4096, 65536, 2 << 20):
    print(f"one, ragged sizes, starts aligned to {al} B", f"{run_ragged(al):.2f} GB/s")
