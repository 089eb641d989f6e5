# One-off probe of the GPU box: host RAM/cores, pinned H2D/D2H bandwidth, HBM size.
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
out["lscpu"] = subprocess.run(["bash","-c","lscpu | grep -E 'Model name|Socket|Core|Thread|NUMA node\\(s\\)'"],capture_output=True,text=True).stdout
free, total = torch.cuda.mem_get_info()
out["hbm_free_total"] = [free, total]
res = {}
for mib in (64, 256, 1024):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    best_h2d = best_d2h = 0
    for _ in range(6):
        with torch.cuda.stream(s):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); d.copy_(h, non_blocking=True); e1.record(s)
        e1.synchronize(); best_h2d = max(best_h2d, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        with torch.cuda.stream(s):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s); h.copy_(d, non_blocking=True); e1.record(s)
        e1.synchronize(); best_d2h = max(best_d2h, n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    res[mib] = (round(best_h2d, 2), round(best_d2h, 2))
out["pinned_gbs_h2d_d2h"] = res
t = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8).pin_memory(); out["pin_8GiB_s"] = time.time() - t
print(json.dumps(out, indent=1))
