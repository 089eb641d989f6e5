"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launches / total / share, as committed under profiles/."""
import csv
import json
import re
import sys
from collections import defaultdict


def main(path, out, command):
    rows = []
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        m = re.search(r"(\w+_kernel(?:<[^()]*>)?)", name)
        key = m.group(1) if m else name[:60]
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r["Metric Unit"], 1e-6)
        rows.append((key, float(r["Metric Value"].replace(",", "")) * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ms in rows:
        agg[k][0] += 1
        agg[k][1] += ms
    total = sum(v[1] for v in agg.values())
    per = [{"kernel": k, "launches": n, "total_ms": round(t, 3),
            "share_pct": round(100 * t / total, 2), "avg_us": round(1e3 * t / n, 2)}
           for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    json.dump({"source": "ncu --metrics gpu__time_duration.sum --clock-control none "
                         "(cold-cache, serialised; compare shares)",
               "command": command, "launches": len(rows), "total_ms": round(total, 3),
               "per_kernel": per}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
