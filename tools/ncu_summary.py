"""Summarise an ncu report (`ncu -i X.ncu-rep --page raw --csv`) into the per-kernel
table kept under profiles/: duration, DRAM bytes read/written, DRAM and SM
throughput, tensor-pipe activity, L2 hit rate, grid, registers.  Optional
--alg NAME=BYTES entries add achieved algorithmic GB/s and the traffic ratio."""
import argparse
import csv
import io
import subprocess

KEYS = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "B"),
        ("dram__bytes_write.sum", "B"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "%"),
        ("lts__t_sector_hit_rate.pct", "%"), ("sm__cycles_elapsed.avg.per_second", "GHz"),
        ("launch__grid_size", ""), ("launch__registers_per_thread", "")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3, "Ghz": 1, "Mhz": 1e-3}

ap = argparse.ArgumentParser()
ap.add_argument("report")
ap.add_argument("--alg", action="append", default=[],
                help="kernel-name-substring=algorithmic bytes per launch")
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units = rows[0], rows[1]
idx = {n: i for i, n in enumerate(head)}
alg = dict(x.split("=", 1) for x in a.alg)
print("kernel | " + " | ".join(k for k, _ in KEYS) + " | alg GB/s | traffic/alg")
for r in rows[2:]:
    name = r[idx["Kernel Name"]]
    vals, num = [], {}
    for k, u in KEYS:
        if k not in idx:
            vals.append("-")
            continue
        v = r[idx[k]].replace(",", "")
        try:
            f = float(v) * SCALE.get(units[idx[k]], 1.0)
        except ValueError:
            vals.append(v)
            continue
        num[k] = f
        vals.append(f"{f:.4g}")
    extra = ""
    for sub, b in alg.items():
        if sub in name and "gpu__time_duration.sum" in num:
            ab = float(b)
            gbs = ab / (num["gpu__time_duration.sum"] * 1e-6) / 1e9
            traffic = num.get("dram__bytes_read.sum", 0) + num.get("dram__bytes_write.sum", 0)
            extra = f" | {gbs:.1f} | {traffic / ab:.3f}"
    print(f"{name[:60]} | " + " | ".join(vals) + extra)
