"""profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each
streaming kernel, from one `ncu --set full` report (bench.py's roofline.traffic).
usage: python tools/make_traffic.py report.ncu-rep [out.json] [config]
The json is keyed by bench config (c2, c1, ...) then kernel; other configs'
entries in an existing file are kept."""
import os
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
config = sys.argv[3] if len(sys.argv) > 3 else "c2"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")
    short = name.split("<")[0].split("(")[0].split()[-1]
    try:
        # the raw page's unit row gives each metric its own unit (byte / Kbyte / Mbyte / Gbyte)
        units = dict(zip(hdr, rows[1]))
        sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = sum(float(d[k].replace(",", "")) * sc.get(units.get(k, "byte"), 1)
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    except (KeyError, ValueError):
        continue
    res.setdefault(short, b)
allres = {}
if os.path.exists(out):
    with open(out) as fh:
        allres = json.load(fh)
    if not all(isinstance(v, dict) for v in allres.values()):
        allres = {}
allres[config] = res
with open(out, "w") as fh:
    json.dump(allres, fh, indent=1)
print(json.dumps(res))
