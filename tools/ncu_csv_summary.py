"""Median per-kernel metric values from an `ncu --csv --log-file` launch list (tuning aid).
usage: python tools/ncu_csv_summary.py FILE.csv"""
import csv
import statistics
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[1:]:
    agg[(r[ki].split("(")[0][-60:], r[mi])].append(float(r[vi].replace(",", "")))
for (k, m), v in sorted(agg.items()):
    print(f"{k:60s} {m:28s} n={len(v):4d} median={statistics.median(v):14.1f}")
