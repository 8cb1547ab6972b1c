"""Static SASS of one kernel from an object/cubin (cuobjdump -sass), with an
opcode histogram -- a quick check of code-generation changes without a GPU.
usage: python tools/sass_fn.py build/fc_run_bf16_a4a4.o <kernel-regex> [--dump out.txt]"""
import collections
import re
import subprocess
import sys

obj, kre = sys.argv[1], sys.argv[2]
dump = sys.argv[sys.argv.index("--dump") + 1] if "--dump" in sys.argv else None
txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", txt)
for f in funcs[1:]:
    name = f.split("\n", 1)[0]
    dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    if not re.search(kre, dem):
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", f)
    ops = collections.Counter()
    for s in ins:
        t = s.split()
        op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        ops[op.split(".")[0]] += 1
    print(dem[:120], "static instructions:", len(ins))
    print("  " + ", ".join(f"{o}:{n}" for o, n in ops.most_common(20)))
    if dump:
        open(dump, "w").write("\n".join(ins))
    break
