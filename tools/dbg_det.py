"""Reduce-only determinism probe: one full call, then the reduce kernel alone (OPT_PHASES 2) on
fixed receive slots, 4 times; the gather slots and outputs must not change."""
import sys; sys.path.insert(0, ".")
import torch
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
tp = 8
m = tp * 8192 * 225
g = torch.Generator(device="cuda").manual_seed(tp)
ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(torch.bfloat16) for r in range(tp)]
for bits in (4, 8):
    cc = fc.CodecConfig(bits=bits); cfg = fc.FlashConfig.uniform(cc)
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, 0)
    for opts in ({}, {_lib.OPT_REDUCE_STAGES: 2}, {_lib.OPT_REDUCE_STAGES: 4}, {_lib.OPT_REDUCE_STAGES: 8},
                 {_lib.OPT_CTAS_PER_SM: 1}, {_lib.OPT_CTAS_PER_SM: 2}, {_lib.OPT_CTAS_PER_SM: 3}):
        comm.set_option(_lib.OPT_PHASES, 0)
        for k, v in opts.items(): comm.set_option(k, v)
        comm.all_reduce_local(ts, cfg)
        comm.set_option(_lib.OPT_PHASES, 2)
        runs = []
        for it in range(4):
            outs = comm.all_reduce_local(ts, cfg)
            runs.append([comm.slot((j + 1) % tp, 2, j, cc).to_bytes() for j in range(tp)])
        print(bits, opts, [runs[i] == runs[0] for i in range(1, 4)], flush=True)
        for k in opts: comm.set_option(k, 0)
    comm.close()
