"""Role timeline of the fused kernel (k_fstream) at C2, all 8 ranks on one GPU:
per role, the window [first start, last end] over CTAs and the mean / max busy
time per CTA, from FC_OPT_ROLE_PROFILE (%globaltimer stamps per CTA).
usage: python tools/fused_profile.py [chunk] [d_stages] [q_stages]"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ds = int(sys.argv[2]) if len(sys.argv) > 2 else 0
qs = int(sys.argv[3]) if len(sys.argv) > 3 else 0
dbg = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # FC_OPT_STREAM_MASK measurement bits (256/512/1024)
tp, M = 8, 8 * 1024 * 8192
cfg = fc.FlashConfig.from_bits(4)
comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
ins = [torch.randn(M, device="cuda").to(torch.bfloat16) for _ in range(tp)]
outs = [torch.empty_like(t) for t in ins]
comm.set_option(_lib.OPT_FUSED, 1)
comm.set_option(_lib.OPT_FUSED_CHUNK, chunk)
comm.set_option(_lib.OPT_GATHER_STAGES, ds)
comm.set_option(_lib.OPT_SCATTER_STAGES, qs)
comm.set_option(_lib.OPT_STREAM_MASK, dbg)
for _ in range(3):
    comm.all_reduce_local(ins, cfg, outs=outs, check=False)
comm.set_option(_lib.OPT_ROLE_PROFILE, 1)
comm.all_reduce_local(ins, cfg, outs=outs, check=dbg & 256 == 0)
torch.cuda.synchronize()
buf = (C.c_uint64 * (4096 * 16))()
n = C.c_int32()
_lib.check(_lib.lib().fc_comm_role_profile(comm._h, 0, buf, 4096, C.byref(n)))
a = np.frombuffer(buf, dtype=np.uint64)[: n.value * 16].reshape(n.value, 16).astype(np.int64)
t0 = a[:, 9].min()
res = {"chunk": chunk, "d_stages": ds, "q_stages": qs, "dbg": dbg, "ctas": n.value,
       "kernel_us": float((a[:, 10].max() - t0) / 1e3), "cta_end_us_min": float((a[:, 10].min() - t0) / 1e3)}
for r, name in enumerate(("scatter", "reduce", "gather")):
    act = a[:, r] > 0
    res[name] = {"first_start_us": float((a[act, r].min() - t0) / 1e3),
                 "last_start_us": float((a[act, r].max() - t0) / 1e3),
                 "first_end_us": float((a[act, 3 + r].min() - t0) / 1e3),
                 "last_end_us": float((a[act, 3 + r].max() - t0) / 1e3),
                 "busy_mean_us": float(a[act, 6 + r].mean() / 1e3), "busy_max_us": float(a[act, 6 + r].max() / 1e3),
                 "ctas": int(act.sum())}
print(json.dumps(res))
comm.close()
