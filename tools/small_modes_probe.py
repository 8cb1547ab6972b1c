"""Small rounds on one GPU: the split phase kernels vs the fused kernel (FC_OPT_FUSED 1) vs
the one-launch small-message kernel (FC_OPT_ONESHOT 2), graph-timed, at C4 bs 8 / 64 and C1."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import graph_time  # noqa: E402

st = torch.cuda.current_stream()
for name, tp, bits, m, dt in (("c4bs8", 8, 4, 8 * 8192, torch.bfloat16), ("c4bs64", 8, 4, 64 * 8192, torch.bfloat16),
                              ("c1", 4, 8, 1024 * 8192, torch.float16)):
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(m, device="cuda").to(dt) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)  # noqa: E731
    comm.set_option(_lib.OPT_FUSED, 0)
    step()
    comm.check()
    ref = [o.clone() for o in outs]
    for mode, opts in (("split", {_lib.OPT_FUSED: 0, _lib.OPT_ONESHOT: 0}),
                       ("fused", {_lib.OPT_FUSED: 1, _lib.OPT_ONESHOT: 0}),
                       ("small", {_lib.OPT_FUSED: 0, _lib.OPT_ONESHOT: 2})):
        for k, v in opts.items():
            comm.set_option(k, v)
        step()
        comm.check()
        ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
        g = graph_time(step, 20, st)
        print(f"{name} {mode}: graph {g*1e3:.1f} us launches {comm.get_option(_lib.OPT_LAST_LAUNCHES)} bitexact {ok}",
              flush=True)
    comm.close()
