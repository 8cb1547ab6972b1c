"""Top stall-sampled SASS lines of one kernel from an ncu source-page CSV.
usage: python tools/src_stalls.py src.csv <kernel-regex> [top]"""
import csv
import re
import sys

path, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
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
    si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_")]
    lines = []
    for r in rr[hdr + 1:]:
        if len(r) <= wi or not r[wi].strip().isdigit():
            continue
        reasons = sorted(((float(r[i] or 0), n[6:]) for i, n in stall_cols if i < len(r) and r[i].replace('.', '', 1).isdigit()), reverse=True)[:2]
        lines.append((int(r[wi]), r[si], reasons))
    tot = sum(n for n, _, _ in lines)
    print(b["name"][:80], "samples", tot)
    for n, s, rs in sorted(lines, key=lambda x: -x[0])[:top]:
        print(f"  {n / tot * 100:5.1f}% {s[:70]:70s} {' '.join(f'{k}:{v:.0f}' for v, k in rs)}")
    break
