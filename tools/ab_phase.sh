#!/bin/bash
# Time one phase kernel of the C2 step (PHASE=1 scatter, 2 reduce, 4 gather) under
# FC_OPT_STREAM_MASK values MASKS (default "0"); outputs checked against mask 0.
cd ${GRAFT_REPO_ROOT:-.}
PHASE=${PHASE:-4} MASKS=${MASKS:-0} python - <<'PY'
import os, sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
phase = int(os.environ["PHASE"]); masks = [int(x) for x in os.environ["MASKS"].split(",")]
tp, m = 8, 8 * 1024 * 8192
cfg = fc.FlashConfig.from_bits(4)
comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
ins = [(torch.randn(m, device="cuda") * (1 + r)).to(torch.bfloat16) for r in range(tp)]
outs = [torch.empty_like(t) for t in ins]
step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
comm.set_option(_lib.OPT_FUSED, 0)
step(); comm.check(); ref = [o.clone() for o in outs]
for mask in masks + masks:
    comm.set_option(_lib.OPT_STREAM_MASK, mask)
    comm.set_option(_lib.OPT_PHASES, 0); step(); comm.check()
    ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
    comm.set_option(_lib.OPT_PHASES, phase)
    for _ in range(3): step()
    ms, _ = _events_time(step, 20, st)
    print(f"phase {phase} mask {mask}: {ms*1e3:.1f} us bitexact {ok}", flush=True)
PY
