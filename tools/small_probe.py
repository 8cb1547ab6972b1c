"""C4 small-message kernel (k_small) timeline: per-CTA first-item start / after-wait / end
(FC_OPT_ROLE_PROFILE), relative to the earliest CTA entry; plus graph latency with and without
the cooperative launch. TP=8 emulated on one GPU."""
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
from bench import graph_time  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
cfg = fc.FlashConfig.from_bits(4)
tp = 8
for bs, warm in ((8, 0), (16, 0)):
    m = bs * 8192
    comm = FlashComm.local([0] * tp, slot_bytes_for(-(-m // tp), cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_ONESHOT, 2)  # the small-message kernel also on one GPU
    ins = [torch.randn(m, device=dev).to(torch.bfloat16) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    res = {}
    for name, mask in (("coop", 0), ("plain", 2048)):
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        res[name] = round(graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), 20, stream) * 1e3, 2)
    comm.check()
    comm.set_option(_lib.OPT_STREAM_MASK, warm)
    comm.set_option(_lib.OPT_ROLE_PROFILE, 1)
    for _ in range(3):
        comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (4096 * 16))()
    n = C.c_int32(0)
    _lib.lib().fc_comm_role_profile(comm._h, 0, buf, 4096, C.byref(n))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16)[: n.value].astype(np.int64)
    t0 = a[:, 0].min()
    out = {"bs": bs, "warm": warm, "graph_us": res, "ctas": int(n.value), "exit_max_us": round((a[:, 5].max() - t0) / 1e3, 2),
           "entry_spread_us": round((a[:, 0].max() - t0) / 1e3, 2)}
    for kind, nm in ((0, "scatter"), (1, "reduce"), (2, "gather")):
        sel = a[a[:, 1] == kind]
        if len(sel):
            out[nm] = {"start": round((sel[:, 2].min() - t0) / 1e3, 2), "wait_done_max": round((sel[:, 3].max() - t0) / 1e3, 2) if kind else None,
                       "end_max": round((sel[:, 4].max() - t0) / 1e3, 2), "dur_med": round(float(np.median(sel[:, 4] - np.where(sel[:, 3] > 0, sel[:, 3], sel[:, 2]))) / 1e3, 2)}
    sel = a[a[:, 1] == 1]
    if len(sel):
        out["reduce_split_us"] = {k: round(float(np.median(sel[:, c1] - sel[:, c0])) / 1e3, 2) for k, c0, c1 in
                                  (("own_qdq", 3, 10), ("src0", 10, 11), ("src1_7", 11, 6), ("sum", 3, 6), ("quant2", 6, 7), ("stores", 7, 8), ("own_out", 8, 9), ("tail", 9, 4))}
    print(json.dumps(out), flush=True)
    comm.set_option(_lib.OPT_ROLE_PROFILE, 0)
    comm.close()
