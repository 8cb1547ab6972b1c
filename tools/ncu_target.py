"""Minimal launch sequence for ncu captures: C2 flash all-reduce (8 logical
ranks on one GPU, fused or split) and C5 quantize/dequantize."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "fused"
tp, M = 8, 8 * 1024 * 8192
if mode.startswith("c4"):  # decode regime: bs x 8192 per rank (c4 -> bs 8, c4_64 -> bs 64)
    M = (int(mode[3:]) if len(mode) > 2 else 8) * 8192
cfg = fc.FlashConfig.from_bits(4)
if mode in ("fused", "split") or mode.startswith("c4"):
    comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, int(mode == "fused"))
    ins = [torch.randn(M, device="cuda").to(torch.bfloat16) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    for _ in range(3):
        comm.all_reduce_local(ins, cfg, outs=outs, check=False)
    comm.check()
else:
    x = torch.randn(M, device="cuda").to(torch.bfloat16)
    if mode.startswith("codec_int"):  # codec_int<bits>_g<group>
        b, g = mode[9:].split("_g")
        cc = fc.CodecConfig(bits=int(b), group_size=int(g))
    else:
        cc = fc.CodecConfig(number_format=mode[6:]) if mode.startswith("codec_") else fc.CodecConfig(bits=4)
    for _ in range(3):
        q = fc.quantize(x, cc)
        fc.dequantize(q, dtype=torch.bfloat16, validate=False)
torch.cuda.synchronize()
