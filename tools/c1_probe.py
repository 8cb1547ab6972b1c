"""C1 (TP=4 INT8 g128 fp16 [1024,8192]) per-phase A/B on one GPU: stream-mask bits,
stage hints and CTA caps; bit-exactness of every variant against the default."""
import itertools
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import _events_time, graph_time  # noqa: E402

st = torch.cuda.current_stream()
tp, bits, m, dt = 4, 8, 1024 * 8192, torch.float16
seg = m // tp
cfg = fc.FlashConfig.from_bits(bits)
comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
ins = [torch.randn(m, device="cuda").to(dt) for _ in range(tp)]
outs = [torch.empty_like(t) for t in ins]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731
comm.set_option(_lib.OPT_FUSED, 0)
comm.set_option(_lib.OPT_PHASES, 0)
step()
comm.check()
ref = [o.clone() for o in outs]


def t(phases, **opts):
    for k, v in opts.items():
        comm.set_option(getattr(_lib, k), v)
    comm.set_option(_lib.OPT_PHASES, 0)
    step()
    comm.check()
    ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
    comm.set_option(_lib.OPT_PHASES, phases)
    for _ in range(3):
        step()
    ms = graph_time(step, 10, st)
    ev, _ = _events_time(step, 30, st)
    for k in opts:
        comm.set_option(getattr(_lib, k), 0)
    comm.set_option(_lib.OPT_PHASES, 0)
    return round(ms * 1e3, 1), round(ev * 1e3, 1), ok


print("step", t(0))
print("step no-PDL", t(0, OPT_STREAM_MASK=8192))
for ph in (1, 2, 4):
    print("phase", ph, "no-PDL", t(ph, OPT_STREAM_MASK=8192))
for ph in (1, 2, 4):
    print("phase", ph, "default", t(ph))
for mask in (16, 64):
    print("scatter mask", mask, t(1, OPT_STREAM_MASK=mask))
for cap in (1, 2, 3, 4):
    print("scatter cap", cap, t(1, OPT_CTAS_PER_SM=cap))
for qs in (2, 3, 6, 8):
    print("scatter qstages", qs, t(1, OPT_SCATTER_STAGES=qs))
for qs, cap in itertools.product((4, 8), (1, 2)):
    print("scatter mask16 qstages", qs, "cap", cap, t(1, OPT_STREAM_MASK=16, OPT_SCATTER_STAGES=qs, OPT_CTAS_PER_SM=cap))
for rs in (2, 3, 6, 8):
    print("reduce stages", rs, t(2, OPT_REDUCE_STAGES=rs))
for cap in (1, 2, 3):
    print("reduce cap", cap, t(2, OPT_CTAS_PER_SM=cap))
for ds in (2, 4, 8, 12):
    print("gather dstages", ds, t(4, OPT_GATHER_STAGES=ds))
for cap in (1, 2, 3, 4):
    print("gather cap", cap, t(4, OPT_CTAS_PER_SM=cap))
