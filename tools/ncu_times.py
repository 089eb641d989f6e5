"""Dev helper: summarise an `ncu --csv --metrics ...` launch list (stdin or a
file) as one line per launch: id, kernel name (shortened), metric values."""
import csv
import sys
from collections import OrderedDict

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
rows = [r for r in csv.reader(src) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
agg = OrderedDict()
for r in rows[1:]:
    agg.setdefault((r[ii], r[ki].split("(")[0][-48:]), {})[r[mi]] = r[vi]
for (i, name), m in agg.items():
    print(i, name, " ".join(f"{k.split('__')[-1]}={v}" for k, v in m.items()))
