"""Key metrics + warp stall breakdown per kernel from an ncu report.
usage: python tools/ncu_summary.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "dram__bytes.sum.peak_sustained": "dram_peak_B/cyc",
    "dram__bytes.sum.per_second": "dram_B/s",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "smsp__inst_executed.sum": "inst",
    "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "launch__grid_size": "grid",
    "lts__t_sector_hit_rate.pct": "l2hit%",
}
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled_") or
              h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if not re.search(kre, d.get("Kernel Name", "")):
        continue
    print(d["Kernel Name"][:70])
    units = dict(zip(hdr, rows[1]))
    sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}

    def val(k):
        x = d.get(k, "?")
        u = units.get(k, "")
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum") and u in sc:  # -> MB
            return f"{float(x.replace(',', '')) * sc[u]:.1f}MB"
        if k == "dram__bytes.sum.per_second" and u.endswith("/s") and u[:-2] in sc:  # -> GB/s
            return f"{float(x.replace(',', '')) * sc[u[:-2]] / 1e3:.0f}GB/s"
        if k == "gpu__time_duration.sum" and u in ("nsecond", "usecond", "msecond"):
            return f"{float(x.replace(',', '')) * {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3}[u]:.1f}us"
        return x
    print("  " + "  ".join(f"{v}={val(k)}" for k, v in keys.items()))
    st = []
    for i in stall_cols:
        try:
            st.append((float(r[i]), hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
    st.sort(reverse=True)
    print("  stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
