#!/bin/bash
# Gather (k_dstream) at C2: CTAs per SM x ring depth sweep.
cd ${GRAFT_REPO_ROOT:-.}
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
for tp, m, bits in ((8, 8 * 1024 * 8192, 4),):
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    comm.set_option(_lib.OPT_FUSED, 0)
    comm.set_option(_lib.OPT_PHASES, 4)
    for cap in (1,):
        for ds in (5, 6, 7, 8):
            comm.set_option(_lib.OPT_CTAS_PER_SM, cap)
            comm.set_option(_lib.OPT_GATHER_STAGES, ds)
            for _ in range(2): step()
            ms, _ = _events_time(step, 10, st)
            print(f"tp{tp} int{bits} cap {cap} stages {ds}: gather {ms*1e3:.1f} us", flush=True)
    comm.close()
PY
