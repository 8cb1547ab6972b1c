"""Executed instructions per CUDA source line (ncu --print-source cuda,sass).
usage: python tools/line_hist.py report.ncu-rep <kernel-regex> <elements> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre, elems = sys.argv[1], sys.argv[2], float(sys.argv[3])
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}", "--launch-count", "1"], capture_output=True, text=True).stdout
cur_file, line_no, line_src = "?", None, ""
acc = collections.Counter()
srcs = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].strip():
        line_no, line_src = r[0], r[1]
        srcs[(cur_file, line_no)] = line_src.strip()[:90]
    ex = r[7] if len(r) > 7 else ""
    if ex.strip().isdigit():
        acc[(cur_file, line_no)] += int(ex)
tot = sum(acc.values())
print("total per elem", round(tot * 32 / elems, 2))
for k, n in acc.most_common(top):
    print(f"{n * 32 / elems:6.2f} {k[0]}:{k[1]:>4} {srcs.get(k, '')}")
