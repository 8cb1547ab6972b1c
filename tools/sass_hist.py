"""Per-opcode executed-instruction histogram of one kernel in an ncu report.
usage: python tools/sass_hist.py report.ncu-rep <kernel-regex> <elements>"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre, elems = sys.argv[1], sys.argv[2], float(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = rows[0][1]
    if not re.search(kre, name):
        continue
    hdr = rows[1]
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_st = hdr.index("Warp Stall Sampling (All Samples)")
    ops, st = collections.Counter(), collections.Counter()
    tot = 0
    for r in rows[2:]:
        if len(r) <= i_ex or not r[i_ex].strip().isdigit():
            continue
        n = int(r[i_ex])
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += n
        st[op] += int(r[i_st] or 0) if r[i_st].strip().isdigit() else 0
        tot += n
    print(name[:80], "warp-instr", tot, "per elem", round(tot * 32 / elems, 2))
    for op, n in ops.most_common(25):
        print(f"  {op:10s} {n * 32 / elems:6.2f}/elem  stall-samples {st[op]}")
    break
