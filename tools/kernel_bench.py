"""Kernel-level timing sweep on one GPU (CUDA events, warm-up, inputs > L2).

  python tools/kernel_bench.py [codec] [flash] [--quick]

codec: C5 quantize / dequantize of bf16 [8,1024,8192] over bits {4,8} x g {32..256}
       (algorithmic bytes (e + b) * M per launch, HBM roofline).
flash: emulated-TP flash all-reduce (fused vs phase-split) at C2 and TP=2/4.
"""

from __future__ import annotations

import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

PEAK = 6550.7


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def codec_sweep(quick=False):
    import ctypes as C

    M = 8 * 1024 * 8192
    x = torch.randn(M, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(M, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    for bits in (4, 8):
        for g in ((128,) if quick else (32, 64, 128, 256)):
            cfg = fc.CodecConfig(bits=bits, group_size=g)
            L = cfg.device_layout(M)
            buf = torch.empty(L.total_bytes, dtype=torch.uint8, device="cuda")
            c = cfg.to_fc()
            q = lambda: _lib.lib().fc_quantize(x.data_ptr(), _lib.DTYPE_BF16, M, C.byref(c), buf.data_ptr(), None, st)
            d = lambda: _lib.lib().fc_dequantize(buf.data_ptr(), M, C.byref(c), out.data_ptr(), _lib.DTYPE_BF16, st)
            tq, td = timeit(q), timeit(d)
            alg = 2 * M + L.wire_bytes
            print(json.dumps({"kernel": "quantize", "bits": bits, "g": g, "us": tq * 1e3,
                              "gbs": alg / tq / 1e6, "frac": alg / tq / 1e6 / PEAK}))
            print(json.dumps({"kernel": "dequantize", "bits": bits, "g": g, "us": td * 1e3,
                              "gbs": alg / td / 1e6, "frac": alg / td / 1e6 / PEAK}))


def flash_sweep(quick=False):
    M = 8 * 1024 * 8192
    e = 2
    cases = [(8, 4)] if quick else [(8, 4), (8, 8), (4, 4), (2, 4)]
    for tp, bits in cases:
        cfg = fc.FlashConfig.from_bits(bits)
        seg = M // tp
        comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
        ins = [torch.randn(M, device="cuda").to(torch.bfloat16) for _ in range(tp)]
        outs = [torch.empty_like(t) for t in ins]
        w = cfg.stage1_codec.wire_byte_len(seg)
        alg = tp * (2 * e * M + 2 * (tp - 1) * 2 * w)
        for mode, opts in (("fused", {}), ("split", {_lib.OPT_FUSED: 0}),
                           ("split_old", {_lib.OPT_FUSED: 0, _lib.OPT_FAST: 2}),
                           ("split_rs2", {_lib.OPT_FUSED: 0, _lib.OPT_REDUCE_STAGES: 2}),
                           ("split_rs3", {_lib.OPT_FUSED: 0, _lib.OPT_REDUCE_STAGES: 3}),
                           ("fused_lag16", {_lib.OPT_LAG: 16})):
            if quick and mode not in ("fused", "split", "split_old", "split_rs2"):
                continue
            comm.set_option(_lib.OPT_FUSED, 1)
            comm.set_option(_lib.OPT_CTAS, 0)
            comm.set_option(_lib.OPT_LAG, 0)
            comm.set_option(_lib.OPT_REDUCE_STAGES, 0)
            comm.set_option(_lib.OPT_FAST, 1)
            for k, v in opts.items():
                comm.set_option(k, v)
            t = timeit(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), iters=10, warm=3)
            comm.check()
            print(json.dumps({"kernel": f"flash_{mode}", "tp": tp, "bits": bits, "ms": t,
                              "alg_gbs": alg / t / 1e6, "frac": alg / t / 1e6 / PEAK,
                              "launches": comm.get_option(_lib.OPT_LAST_LAUNCHES)}))
        comm.close()
        del ins, outs
        torch.cuda.empty_cache()


def tune_sweep():
    """Ring depths / CTA caps of the streaming split kernels at C2 (8 logical ranks)."""
    M, tp, e = 8 * 1024 * 8192, 8, 2
    cfg = fc.FlashConfig.from_bits(4)
    seg = M // tp
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, 0)
    ins = [torch.randn(M, device="cuda").to(torch.bfloat16) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    w = cfg.stage1_codec.wire_byte_len(seg)
    alg = tp * (2 * e * M + 2 * (tp - 1) * 2 * w)
    grid = [dict()]
    grid += [{_lib.OPT_SCATTER_STAGES: q} for q in (2, 3, 6, 8)]
    grid += [{_lib.OPT_GATHER_STAGES: d} for d in (3, 4, 8, 12)]
    grid += [{_lib.OPT_REDUCE_STAGES: r} for r in (1, 3, 4)]
    grid += [{_lib.OPT_CTAS_PER_SM: c} for c in (1, 2, 3)]
    # per phase; stream-mask bits 6/7: the 32-element-lane INT4 g128 scatter / reduce (A/B)
    grid += [{_lib.OPT_PHASES: 1}, {_lib.OPT_PHASES: 1, _lib.OPT_STREAM_MASK: 64},
             {_lib.OPT_PHASES: 2}, {_lib.OPT_PHASES: 2, _lib.OPT_STREAM_MASK: 128},
             {_lib.OPT_PHASES: 4}]
    for opts in grid:
        for o in (_lib.OPT_SCATTER_STAGES, _lib.OPT_GATHER_STAGES, _lib.OPT_REDUCE_STAGES, _lib.OPT_CTAS_PER_SM,
                  _lib.OPT_STREAM_MASK, _lib.OPT_PHASES):
            comm.set_option(o, 0)
        for k, v in opts.items():
            comm.set_option(k, v)
        t = timeit(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), iters=10, warm=3)
        comm.check()
        print(json.dumps({"kernel": "flash_split_tune", "opts": {str(k): v for k, v in opts.items()}, "ms": t,
                          "frac": alg / t / 1e6 / PEAK}))
    comm.close()


def fused_tune():
    """Schedule chunk / ring depths / CTA cap of the fused streaming kernel at C2
    (all 8 ranks in one launch), against the phase-split path."""
    M, tp, e = 8 * 1024 * 8192, 8, 2
    cfg = fc.FlashConfig.from_bits(4)
    seg = M // tp
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    ins = [torch.randn(M, device="cuda").to(torch.bfloat16) for _ in range(tp)]
    outs = [torch.empty_like(t) for t in ins]
    w = cfg.stage1_codec.wire_byte_len(seg)
    alg = tp * (2 * e * M + 2 * (tp - 1) * 2 * w)
    comm.set_option(_lib.OPT_FUSED, 0)
    t = timeit(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), iters=10, warm=3)
    print(json.dumps({"kernel": "flash_split", "ms": t, "frac": alg / t / 1e6 / PEAK}), flush=True)
    comm.set_option(_lib.OPT_FUSED, 1)
    tiles = seg // 8192
    for chunk in (0, tiles // 4):
        for qs, ds, cap, gc, rs in ((0, 0, 0, 0, 0), (4, 4, 0, 0, 0), (4, 8, 0, 0, 0), (6, 0, 0, 0, 0),
                                    (0, 0, 0, 1, 0), (0, 6, 0, 1, 0), (0, 0, 0, 2, 0), (4, 0, 2, 0, 0),
                                    (0, 0, 0, 0, 6), (0, 0, 0, 0, 12), (0, 0, 0, 0, 16), (8, 0, 0, 0, 16)):
            comm.set_option(_lib.OPT_REDUCE_STAGES, rs)
            comm.set_option(_lib.OPT_FUSED_CHUNK, chunk)
            comm.set_option(_lib.OPT_SCATTER_STAGES, qs)
            comm.set_option(_lib.OPT_GATHER_STAGES, ds)
            comm.set_option(_lib.OPT_CTAS_PER_SM, cap)
            comm.set_option(_lib.OPT_FUSED_GATHER_CTAS, gc)
            t = timeit(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), iters=10, warm=3)
            comm.check()
            print(json.dumps({"kernel": "flash_fused_tune", "chunk": chunk, "q_stages": qs, "d_stages": ds,
                              "cta_cap": cap, "gather_ctas_per_sm": gc, "r_ring": rs, "ms": t, "frac": alg / t / 1e6 / PEAK}),
                  flush=True)
    comm.close()


if __name__ == "__main__":
    what = [a for a in sys.argv[1:] if not a.startswith("--")] or ["codec", "flash"]
    quick = "--quick" in sys.argv
    if "codec" in what:
        codec_sweep(quick)
    if "flash" in what:
        flash_sweep(quick)
    if "tune" in what:
        tune_sweep()
    if "fusedtune" in what:
        fused_tune()
