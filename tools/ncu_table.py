"""Summarise an `ncu --csv --metrics ...` log: mean of each metric per kernel
(short name). Usage: python tools/ncu_table.py log.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
acc = defaultdict(lambda: defaultdict(list))
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    try:
        acc[name][r[-3]].append(float(r[-1].replace(",", "")))
    except ValueError:
        pass
for k, m in acc.items():
    print(k)
    for metric, v in m.items():
        print(f"   {metric:60s} {sum(v) / len(v):14.1f}  (n={len(v)})")
