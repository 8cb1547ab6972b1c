#!/bin/bash
# A/B of the reduce kernel: 2-lanes-per-group INT4 g128 (default for whole tiles) vs the
# 32-element lane layout (FC_OPT_STREAM_MASK bit 7); bit-exactness checked against the old kernel.
cd ${GRAFT_REPO_ROOT:-.}
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
for tp, m, dt, cfg in ((4, 1024 * 8192, torch.float16, fc.FlashConfig.from_bits(8)),
                       (8, 8 * 1024 * 8192, torch.bfloat16, fc.FlashConfig.from_bits(8)),
                       (8, 8 * 1024 * 8192, torch.bfloat16, fc.FlashConfig.from_bits(4)),
                       (4, 8 * 1024 * 8192, torch.float16, fc.FlashConfig.from_bits(4)),
                       (8, 8 * 1024 * 8192, torch.bfloat16,
                        fc.FlashConfig.uniform(fc.CodecConfig(bits=4, symmetric=True))), (8, 8 * 1024 * 8192, torch.bfloat16, fc.FlashConfig.uniform(fc.CodecConfig(bits=4, rounding="ceil")))):
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    ins = [(torch.randn(m, device="cuda") * (1 + r)).to(dt) for r in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    comm.set_option(_lib.OPT_FUSED, 0)
    comm.set_option(_lib.OPT_STREAM_MASK, 128)
    step(); comm.check(); ref = [o.clone() for o in outs]
    for mask in (0, 128, 0):
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        comm.set_option(_lib.OPT_PHASES, 0); step(); comm.check()
        ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
        comm.set_option(_lib.OPT_PHASES, 2)
        for _ in range(3): step()
        ms, _ = _events_time(step, 20, st)
        print(f"tp{tp} {dt} int{cfg.stage1_codec.bits} sym={cfg.stage1_codec.symmetric} mask {mask}: reduce {ms*1e3:.1f} us bitexact {ok}", flush=True)
    comm.close()
PY
