"""Bitwise A/B of the split kernels at TP=8 (8 logical ranks, 1 GPU): every
mix of streaming vs staged scatter/reduce/gather against the staged path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2412_04964_b200 as fc
from paper_2412_04964_b200 import _lib
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

for bits in (8, 4):
    for M in (1024 * 8192, 65536 * 8 * 3):
        tp = 8
        cfg = fc.FlashConfig.from_bits(bits)
        comm = FlashComm.local([0] * tp, slot_bytes_for(-(-M // tp), cfg.stage1_codec, cfg.stage2_codec))
        comm.set_option(_lib.OPT_FUSED, 0)
        g = torch.Generator(device="cuda").manual_seed(7)
        ins = [torch.randn(M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(tp)]
        comm.set_option(_lib.OPT_FAST, 2)
        ref = [o.clone() for o in comm.all_reduce_local(ins, cfg, out_dtype=torch.float32)]
        comm.set_option(_lib.OPT_FAST, 1)
        for mask in range(8):
            comm.set_option(_lib.OPT_STREAM_MASK, mask)
            outs = comm.all_reduce_local(ins, cfg, out_dtype=torch.float32)
            bad = [r for r in range(tp) if not torch.equal(outs[r].view(torch.int32), ref[r].view(torch.int32))]
            nbad = sum(int((outs[r].view(torch.int32) != ref[r].view(torch.int32)).sum()) for r in bad)
            print(f"bits={bits} M={M} mask={mask} (1=staged scatter,2=staged reduce,4=staged gather) bad_ranks={bad} bad_elems={nbad}", flush=True)
        comm.close()
