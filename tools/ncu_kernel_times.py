"""Average gpu__time_duration per kernel name from an ncu --csv metrics dump on stdin."""
import collections
import csv
import sys

rows = [l for l in sys.stdin if not l.startswith("==")]
r = csv.reader(rows)
h = next(r)
d = collections.defaultdict(list)
for row in r:
    row = dict(zip(h, row))
    if row.get("Metric Name") == "gpu__time_duration.sum":
        d[row["Kernel Name"][:60]].append(float(row["Metric Value"].replace(",", "")))
for k, v in d.items():
    print(f"{k:60s} n={len(v):4d} avg={sum(v) / len(v):10.1f} {row.get('Metric Unit', '')}")
