"""Small launch sequence for compute-sanitizer (racecheck / synccheck / memcheck):
TP=8 INT4 and INT8 g128 flash all-reduce of bf16 (8 logical ranks on cuda:0,
6 tiles per segment so every CTA ring wraps), phase-split (k_qstream_gpl /
k_rstream_gpl / k_dstream) or fused (k_fstream, chunked schedule), and the
single-GPU codec; lane8: the minifloat / rotation paths. Checks the result against the split path bit for bit.
usage: python tools/sanitize_target.py split|fused|codec|small|lane8"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "split"
tp, M = 8, 8 * 8192 * 6
g = torch.Generator(device="cuda").manual_seed(5)
ins = [torch.randn(M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(tp)]
if mode in ("split", "fused"):
    for bits, odt in ((4, torch.bfloat16), (8, torch.bfloat16), (4, torch.float32)):  # fp32: the register-direct reduce output
        cfg = fc.FlashConfig.from_bits(bits)
        comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
        comm.set_timeout(1200.0)  # racecheck slows the flag-synchronised kernels by 100-1000x
        comm.set_option(_lib.OPT_FUSED, 0)
        ref = [o.clone() for o in comm.all_reduce_local(ins, cfg, out_dtype=odt)]
        comm.set_option(_lib.OPT_FUSED, int(mode == "fused"))
        if mode == "fused":
            comm.set_option(_lib.OPT_FUSED_CHUNK, 2)
        for _ in range(2):
            outs = comm.all_reduce_local(ins, cfg, out_dtype=odt)
        assert all(torch.equal(a, b) for a, b in zip(outs, ref)), mode
        comm.close()
elif mode == "small":  # decode-sized rounds: the one-launch k_small (vs the split kernels)
    for bits in (4, 8):
        cfg = fc.FlashConfig.from_bits(bits)
        ms = 8 * 8192 * 2
        sins = [t[:ms].contiguous() for t in ins]
        comm = FlashComm.local([0] * tp, slot_bytes_for(ms // tp, cfg.stage1_codec, cfg.stage2_codec))
        comm.set_option(_lib.OPT_ONESHOT, 0)
        ref = [o.clone() for o in comm.all_reduce_local(sins, cfg)]
        comm.set_option(_lib.OPT_ONESHOT, 2)  # the small-message kernel also on one GPU
        for _ in range(2):
            outs = comm.all_reduce_local(sins, cfg)
        assert all(torch.equal(a.view(torch.int16), b.view(torch.int16)) for a, b in zip(outs, ref)), mode
        comm.close()
elif mode == "lane8":  # minifloat stages and the fused rotation (k_l8_*), plus the minifloat codec
    for cfg in (fc.FlashConfig.uniform(fc.CodecConfig(number_format="e4m3")),
                fc.FlashConfig(fc.CodecConfig(bits=4), fc.CodecConfig(bits=4), rotation=fc.HadamardBlock(128, sign_seed=3))):
        comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
        for _ in range(2):
            fc.flash_all_reduce(ins, cfg, comm=comm, out_dtype=torch.float32)
        comm.close()
    # minifloat stages with bf16 outputs: the streaming kernels on MfSpec, against the lane-8 ones
    for f in ("e4m3", "e2m1"):
        cfg = fc.FlashConfig.uniform(fc.CodecConfig(number_format=f))
        comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
        comm.set_option(_lib.OPT_STREAM_MASK, 1024)
        ref = [o.clone() for o in comm.all_reduce_local(ins, cfg)]
        comm.set_option(_lib.OPT_STREAM_MASK, 0)
        for _ in range(2):
            outs = comm.all_reduce_local(ins, cfg)
        assert all(torch.equal(a.view(torch.int16), b.view(torch.int16)) for a, b in zip(outs, ref)), f
        comm.close()
    for f in ("e4m3", "e2m1"):
        q = fc.quantize(ins[0], fc.CodecConfig(number_format=f))
        fc.dequantize(q, dtype=torch.bfloat16)
else:
    for bits in (4, 8):
        q = fc.quantize(ins[0], fc.CodecConfig(bits=bits))
        fc.dequantize(q, dtype=torch.bfloat16)
torch.cuda.synchronize()
print("ok", mode)
