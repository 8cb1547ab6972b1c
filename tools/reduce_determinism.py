"""Reduce-only determinism probe: one full flash all-reduce, then the reduce kernel alone (OPT_PHASES 2)
on fixed receive slots 4 times; the stage-2 gather slots must not change. It caught the INT8-sym
ring-slot release race. usage: python tools/reduce_determinism.py TP sym|asym [special]"""
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
tp = int(sys.argv[1]); bits = 8; sym = sys.argv[2] == "sym"
m = tp * 8192 * (-(-1800 // tp))
cc = fc.CodecConfig(bits=bits, symmetric=sym); cfg = fc.FlashConfig.uniform(cc)
comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
comm.set_option(_lib.OPT_FUSED, 0)
g = torch.Generator(device="cuda").manual_seed(tp)
ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(torch.bfloat16) for r in range(tp)]
if "special" in sys.argv:
    ts[0][5000:5128] = 1000.0
    ts[1][9000:9128] += 3000.0
comm.all_reduce_local(ts, cfg)

comm.set_option(_lib.OPT_PHASES, 2)  # the reduce alone, on fixed receive slots
runs = []
for it in range(4):
    outs = comm.all_reduce_local(ts, cfg)
    runs.append([comm.slot((j + 1) % tp, 2, j, cc).to_bytes() for j in range(tp)])
print(sys.argv[1:], "reduce-only runs identical:", [runs[i] == runs[0] for i in range(4)], flush=True)
import numpy as np
seg = m // tp
for i in range(1, 4):
    for j in range(tp):
        a = np.frombuffer(runs[0][j], np.uint8); b = np.frombuffer(runs[i][j], np.uint8)
        d = np.nonzero(a != b)[0]
        if len(d):
            cb = seg * bits // 8
            dc = d[d < cb]
            lanes = np.unique(dc // 64)  # INT8: 64 code bytes per lane
            print(f"run{i} owner{j}: {len(dc)} code bytes, {len(d) - len(dc)} meta bytes; tiles {np.unique(dc // 8192)[:8].tolist()} lanes-in-tile {np.unique((dc % 8192) // 64)[:40].tolist()}")
            off = dc[0]
            print("    run0", a[off:off+16].tolist(), "run_i", b[off:off+16].tolist())
            break
