"""Opcode histogram + hottest SASS lines per kernel from an ncu source-page CSV
(ncu -i rep --page source --csv --print-source sass).
usage: python tools/src_hist.py src.csv <kernel-regex> <elements> [lines]"""
import collections
import csv
import re
import sys

path, kre, elems = sys.argv[1], sys.argv[2], float(sys.argv[3])
nl = int(sys.argv[4]) if len(sys.argv) > 4 else 0
rows = list(csv.reader(open(path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if cur is not None:
        cur["rows"].append(r)
for b in blocks:
    if not re.search(kre, b["name"]):
        continue
    rr = b["rows"]
    hdr = next(i for i, r in enumerate(rr) if "Source" in r and "Instructions Executed" in r)
    h = rr[hdr]
    si, ei = h.index("Source"), h.index("Instructions Executed")
    lines = [(int(r[ei]), r[si]) for r in rr[hdr + 1:] if len(r) > ei and r[ei].strip().isdigit()]
    tot = sum(n for n, _ in lines)
    ops = collections.Counter()
    for n, s in lines:
        t = s.split()
        if t:
            op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
            ops[op.split(".")[0]] += n
    print(b["name"][:90], "warp-instr", tot, "per elem", round(tot * 32 / elems, 2))
    print("  " + ", ".join(f"{o}:{n * 32 / elems:.2f}" for o, n in ops.most_common(24)))
    if nl:
        mx = max(n for n, _ in lines)
        for n, s in lines:
            if n >= mx * 0.5:
                print(f"   {n / mx:4.2f} {s[:96]}")
    break
