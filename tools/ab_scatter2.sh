#!/bin/bash
# Scatter A/B: group-per-lane with staged coalesced code stores (mask 0 / 16 for INT8),
# direct strided stores (32 / 48), the 32-element lanes (64); bit-exactness vs the lanes kernel.
cd ${GRAFT_REPO_ROOT:-.}
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
for tp, bits, m, dt, masks in ((8, 4, 8 * 1024 * 8192, torch.bfloat16, (0, 32, 64)),
                                (8, 8, 8 * 1024 * 8192, torch.bfloat16, (16, 48, 64)),
                                (4, 8, 1024 * 8192, torch.float16, (16, 48, 64))):
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(m, device="cuda").to(dt) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    comm.set_option(_lib.OPT_FUSED, 0)
    comm.set_option(_lib.OPT_STREAM_MASK, 64 | 128); step(); comm.check(); ref = [o.clone() for o in outs]
    for mask in masks + masks:
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        comm.set_option(_lib.OPT_PHASES, 0); step(); comm.check()
        ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
        comm.set_option(_lib.OPT_PHASES, 1)
        for _ in range(3): step()
        ms, _ = _events_time(step, 20, st)
        print(f"tp{tp} int{bits} mask {mask}: scatter {ms*1e3:.1f} us bitexact {ok}", flush=True)
    comm.close()
PY
