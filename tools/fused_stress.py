"""Bitwise stress of the fused kernel (k_fstream) against the phase-split path on one GPU:
TP=8 / 4, INT4 / INT8 asym and sym g128, bf16, schedule chunks 1 / 2 / auto, many calls.
usage: python tools/fused_stress.py [iterations]"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad_total = 0
for tp in (8, 4):
    m = tp * 8192 * 48
    g = torch.Generator(device="cuda").manual_seed(tp)
    ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(torch.bfloat16) for r in range(tp)]
    for cc in (fc.CodecConfig(bits=4), fc.CodecConfig(bits=8), fc.CodecConfig(bits=4, symmetric=True),
               fc.CodecConfig(bits=8, symmetric=True)):
        cfg = fc.FlashConfig.uniform(cc)
        comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
        comm.set_option(_lib.OPT_FUSED, 0)
        ref = [o.clone() for o in comm.all_reduce_local(ts, cfg)]
        comm.set_option(_lib.OPT_FUSED, 1)
        for chunk in (1, 2, 0):
            comm.set_option(_lib.OPT_FUSED_CHUNK, chunk)
            bad = 0
            for _ in range(iters):
                outs = comm.all_reduce_local(ts, cfg, check=False)
                bad += sum(int((a.view(torch.int16) != b.view(torch.int16)).sum()) for a, b in zip(outs, ref))
            comm.check()
            bad_total += bad
            print(f"tp={tp} bits={cc.bits} sym={cc.symmetric} chunk={chunk}: {iters} calls, mismatching elements {bad}", flush=True)
        comm.close()
print("TOTAL mismatches", bad_total)
