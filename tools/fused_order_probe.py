"""Fused vs split at C2 on one comm, in alternating order (events, 20 steps each), to
separate the kernels' own times from measurement-order effects in the bench line."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import _events_time, graph_time  # noqa: E402

st = torch.cuda.current_stream()
tp, m = 8, 8 * 1024 * 8192
cfg = fc.FlashConfig.from_bits(4)
comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
ins = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(tp)]
outs = [torch.empty_like(t) for t in ins]
step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731
for mode in ("fused", "split", "fused", "split", "fused"):
    comm.set_option(_lib.OPT_FUSED, 1 if mode == "fused" else 0)
    for _ in range(2):
        step()
    ev, per = _events_time(step, 20, st)
    comm.check()
    g = graph_time(step, 10, st)
    print(f"{mode}: events {ev*1e3:.1f} us (min {min(per)*1e3:.1f} max {max(per)*1e3:.1f})  graph {g*1e3:.1f} us", flush=True)
