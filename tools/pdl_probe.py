"""Programmatic dependent launch A/B (FC_OPT_STREAM_MASK bit 13 = plain launches) of the
phase-split streaming kernels: C2, C1 and C4 (bs 8 / 64) steps, graph- and event-timed."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import _events_time, graph_time  # noqa: E402

st = torch.cuda.current_stream()
for name, tp, bits, m, dt in (("c2", 8, 4, 8 * 1024 * 8192, torch.bfloat16), ("c1", 4, 8, 1024 * 8192, torch.float16),
                              ("c4bs8", 8, 4, 8 * 8192, torch.bfloat16), ("c4bs64", 8, 4, 64 * 8192, torch.bfloat16)):
    seg = m // tp
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(m, device="cuda").to(dt) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731
    step()
    comm.check()
    ref = [o.clone() for o in outs]
    for mask in (0, 8192, 0, 8192):
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        step()
        comm.check()
        ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
        for _ in range(3):
            step()
        g = graph_time(step, 20, st)
        ev, _ = _events_time(step, 30, st)
        comm.check()
        print(f"{name} mask {mask}: graph {g*1e3:.1f} us events {ev*1e3:.1f} us launches "
              f"{comm.get_option(_lib.OPT_LAST_LAUNCHES)} bitexact {ok}", flush=True)
    comm.close()
