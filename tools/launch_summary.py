"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv`):
launches, average duration and share of this package's kernels per kernel.
usage: python tools/launch_summary.py launches.csv [header line]"""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
per = collections.OrderedDict()
for r in rows:
    name, ns = r[4], float(r[14].replace(",", ""))
    per.setdefault(name, []).append(ns)
ours = sum(sum(v) for k, v in per.items() if "fc::" in k)
if len(sys.argv) > 2:
    print(sys.argv[2])
for name, v in per.items():
    share = f"{100 * sum(v) / ours:5.1f}%" if "fc::" in name and ours else "   - "
    print(f"{len(v):4d} launches  avg {sum(v) / len(v) / 1e3:9.1f} us  share of fc kernels {share}  {name[:100]}")
