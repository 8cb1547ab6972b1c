"""TP=2/4/8 INT4 / INT8 g128 at 64 Mi elements per rank: the group-lane reduce with the own piece
through the slots (default, ownq) vs the 32-element-lane reduce that QDQs the own piece in
registers (FC_OPT_STREAM_MASK bit 7), graph-timed, bit-exact against each other."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import graph_time  # noqa: E402

st = torch.cuda.current_stream()
m = 64 << 20
for tp in (2, 4, 8):
    for bits in (4, 8):
        cfg = fc.FlashConfig.from_bits(bits)
        comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
        ins = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(tp)]
        outs = [torch.empty_like(t) for t in ins]
        step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731
        comm.set_option(_lib.OPT_FUSED, 0)
        res = {}
        for mask in (0, 128):
            comm.set_option(_lib.OPT_STREAM_MASK, mask)
            step()
            comm.check()
            res[mask] = ([o.clone() for o in outs], graph_time(step, 5, st))
        ok = all(torch.equal(a, b) for a, b in zip(res[0][0], res[128][0]))
        print(f"tp{tp} int{bits}: ownq+gpl {res[0][1]*1e3:.1f} us  lane32 {res[128][1]*1e3:.1f} us  bitexact {ok}",
              flush=True)
        comm.close()
        del ins, outs, res
        torch.cuda.empty_cache()
