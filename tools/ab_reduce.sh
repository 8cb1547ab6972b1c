#!/bin/bash
# A/B of the reduce kernel's ring depth (FC_OPT_REDUCE_STAGES) at C2; bit-exactness checked.
cd ${GRAFT_REPO_ROOT:-.}
C1=${C1:-} python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
import os
tp, m, bits = (4, 1024 * 8192, 8) if os.environ.get("C1") else (8, 8 * 1024 * 8192, 4)
cfg = fc.FlashConfig.from_bits(bits)
comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
ins = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(tp)]
outs = [torch.empty_like(t) for t in ins]
step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
comm.set_option(_lib.OPT_FUSED, 0)
step(); comm.check(); ref = [o.clone() for o in outs]
for stages in (0, 1, 2, 1, 0):
    comm.set_option(_lib.OPT_REDUCE_STAGES, stages)
    comm.set_option(_lib.OPT_PHASES, 0); step(); comm.check()
    ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
    comm.set_option(_lib.OPT_PHASES, 2)
    for _ in range(3): step()
    ms, _ = _events_time(step, 20, st)
    print(f"reduce stages {stages}: {ms*1e3:.1f} us bitexact {ok}", flush=True)
PY
