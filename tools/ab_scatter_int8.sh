#!/bin/bash
# A/B of the scatter kernel: group-per-lane (default at g=128) vs the 32-element lane layout
# (FC_OPT_STREAM_MASK bit 64; MASKB=16: INT8 on the group-per-lane kernel), per config: TP, bits, elements per rank. Bit-exactness checked.
cd ${GRAFT_REPO_ROOT:-.}
python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for
from bench import _events_time
st = torch.cuda.current_stream()
for tp, bits, m, dt in ((8, 4, 8 * 1024 * 8192, torch.bfloat16), (4, 8, 1024 * 8192, torch.float16),
                        (8, 8, 8 * 1024 * 8192, torch.bfloat16)):
    seg = m // tp
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(m, device="cuda").to(dt) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    step = lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    comm.set_option(_lib.OPT_FUSED, 0)
    res = {}
    for mask in (0, 16, 0, 16):
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        comm.set_option(_lib.OPT_PHASES, 0); step(); comm.check()
        if mask == 0 and 0 not in res:
            ref = [o.clone() for o in outs]
        ok = all(torch.equal(o, r) for o, r in zip(outs, ref))
        comm.set_option(_lib.OPT_PHASES, 1)
        for _ in range(3): step()
        ms, _ = _events_time(step, 20, st)
        res[mask] = ms
        print(f"tp{tp} int{bits} m={m} mask {mask}: scatter {ms*1e3:.1f} us bitexact {ok}", flush=True)
    comm.close()
PY
