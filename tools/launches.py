"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count/mean/min/max (us)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in data:
    agg[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")) / 1e3)
tot = sum(sum(v) for k, v in agg.items() if "sa::" in k)
print(f"{'kernel':48s} {'n':>5s} {'mean_us':>9s} {'min_us':>9s} {'max_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = sum(v) / tot if "sa::" in k else float("nan")
    print(f"{k:48s} {len(v):5d} {sum(v)/len(v):9.2f} {min(v):9.2f} {max(v):9.2f} {share:6.1%}")
