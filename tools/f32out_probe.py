"""fp32 outputs (the reference's output dtype) at C2: the group-lane reduce (default) vs the
32-element-lane reduce (FC_OPT_STREAM_MASK bit 7), INT4 and e4m3 stages, graph-timed, bit-exact."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402
from bench import graph_time  # noqa: E402

st = torch.cuda.current_stream()
tp, m = 8, 8 * 1024 * 8192
ins = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(tp)]
outs = [torch.empty(m, device="cuda", dtype=torch.float32) for _ in range(tp)]
for name, cfg, masks in (("int4", fc.FlashConfig.from_bits(4), (0, 128)),
                         ("e4m3", fc.FlashConfig.uniform(fc.CodecConfig(number_format="e4m3")), (0, 1024))):
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, 0)
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, out_dtype=torch.float32, check=False)  # noqa: E731
    res = {}
    for mask in masks:
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        step()
        comm.check()
        res[mask] = ([o.clone() for o in outs], graph_time(step, 5, st))
    ok = all(torch.equal(a, b) for a, b in zip(res[masks[0]][0], res[masks[1]][0]))
    print(f"{name} fp32 out: default {res[masks[0]][1]*1e3:.1f} us  mask {masks[1]} {res[masks[1]][1]*1e3:.1f} us  "
          f"bitexact {ok}", flush=True)
    comm.close()
    del res
    torch.cuda.empty_cache()
