"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum); dev tool.
usage: python tools/kernel_times.py LAUNCHES.csv [divide_by]"""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    n, t = agg.get(r[ik], (0, 0.0))
    agg[r[ik]] = (n + 1, t + v)
tot = sum(t for _, t in agg.values())
for k, (n, t) in agg.items():
    print(f"{k[:48]:48s} launches {n:5d}  ms {t / 1e6 / div:9.3f}  share {t / tot * 100:5.1f}%")
