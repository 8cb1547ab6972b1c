"""Phase-time sweep of the C2 flash all-reduce on one GPU (8 logical ranks):
each phase alone (OPT_PHASES) under a few option settings.
usage: python tools/reduce_probe.py [bits] [dtype] ; env SWEEP='opt=val,opt=val;...'"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tp = int(os.environ.get("TP", "8"))
M = int(os.environ.get("M", str(8 * 1024 * 8192)))
cfg = fc.FlashConfig.from_bits(bits)
comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
comm.set_option(_lib.OPT_FUSED, 0)
g = torch.Generator(device="cuda").manual_seed(1)
ins = [torch.randn(M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(tp)]
outs = [torch.empty_like(t) for t in ins]
step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731


def timeit(n=20):
    for _ in range(3):
        step()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


names = {k[4:].lower(): getattr(_lib, k) for k in dir(_lib) if k.startswith("OPT_")}
for setting in os.environ.get("SWEEP", "").split(";"):
    opts = [kv.split("=") for kv in setting.split(",") if kv]
    for k, v in opts:
        comm.set_option(names[k], int(v))
    res = {}
    for bit, nm in ((0, "step"), (1, "scatter"), (2, "reduce"), (4, "gather")):
        comm.set_option(_lib.OPT_PHASES, bit)
        res[nm] = round(timeit(), 1)
    comm.set_option(_lib.OPT_PHASES, 0)
    comm.check()
    print(f"bits={bits} tp={tp} [{setting}] " + " ".join(f"{k}={v}" for k, v in res.items()), flush=True)
    for k, v in opts:
        comm.set_option(names[k], 0 if k != "fused" else -1)
