"""Mean duration and warp instructions per kernel from an ncu --csv metric
dump on stdin (gpu__time_duration.sum, smsp__inst_executed.sum)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(sys.stdin) if r]
hi = [i for i, r in enumerate(rows) if r[0] == "ID"]
if not hi:
    sys.exit("no ncu table on stdin")
h = rows[hi[0]]
agg = collections.defaultdict(list)
for r in rows[hi[0] + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    agg[(d["Kernel Name"].split("(")[0], d["Metric Name"])].append(float(d["Metric Value"].replace(",", "")))
for (k, m), v in sorted(agg.items()):
    print(f"{k[:60]:60s} {m:28s} n={len(v):4d} mean={sum(v) / len(v):.1f}")
