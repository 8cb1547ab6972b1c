"""profiles/<round>_sass_evidence.txt: for each hot kernel of the C2 path (bf16,
INT4 g128), the static SASS counts of the instructions that prove the
Blackwell data movement -- UBLKCP (cp.async.bulk: the TMA engine's bulk
copy), SYNCS (mbarrier arrive/wait), plus the packed fp32x2 math -- and a short
excerpt around the first bulk copy.
usage: python tools/sass_evidence.py paper_2412_04964_b200/csrc/build/fc_run_bf16_a4a4.o > out.txt"""
import collections
import re
import subprocess
import sys

obj = sys.argv[1]
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
want = ("k_qstream_gpl", "k_rstream_gpl", "k_dstream", "k_fstream")
print(f"# cuobjdump -sass {obj} (sm_100a)")
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n", 1)[0]
    dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    short = dem.split("<")[0].split()[-1].split("::")[-1]
    if short not in want or "__nv_bfloat16" not in dem:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", f)
    ops = collections.Counter()
    for s in ins:
        t = s.split()
        op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        ops[op] += 1
    key = {k: sum(v for o, v in ops.items() if o.startswith(k)) for k in
           ("UBLKCP", "SYNCS", "FFMA2", "FMUL2", "FADD2", "PRMT", "LDS", "STG", "LDG", "RED", "ST.E", "LD.E")}
    print(f"\n== {dem[:160]}\n   static instructions: {len(ins)}")
    print("   " + ", ".join(f"{k}:{v}" for k, v in key.items()))
    first = next((i for i, s in enumerate(ins) if "UBLKCP" in s), None)
    if first is not None:
        print("   excerpt:")
        for s in ins[max(0, first - 3): first + 4]:
            print("     " + s.strip())
    syncs = sorted({s.split()[0] if not s.startswith("@") else s.split()[1] for s in ins if "SYNCS" in s})
    print("   SYNCS forms: " + ", ".join(syncs))
