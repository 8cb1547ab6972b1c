"""End-to-end (host-buffer) path probe: where the time of
fc_flash_all_reduce_host goes at the bench configuration -- pinned output
allocation, chunk size sweep, against plain pinned H2D / D2H copies.

usage: python tools/e2e_probe.py [--config c2]
"""

from __future__ import annotations

import argparse
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from bench import CONFIGS, _dtype  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402


def wall(fn, reps=3):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    tp, dt, m = cfg["tp"], _dtype(cfg["dtype"]), math.prod(cfg["shape"])
    seg = -(-m // tp)
    fcfg = fc.FlashConfig.from_bits(cfg["bits"], group_size=cfg["group"])
    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, fcfg.stage1_codec, fcfg.stage2_codec))
    hs = [torch.randn(m).to(dt).pin_memory() for _ in range(tp)]
    ds = [torch.empty(m, dtype=dt, device="cuda") for _ in range(tp)]
    print(f"alloc pinned outputs: {wall(lambda: [torch.empty(m, dtype=dt, pin_memory=True) for _ in range(tp)]):.2f} ms")
    print(f"H2D only: {wall(lambda: [d.copy_(h, non_blocking=True) for h, d in zip(hs, ds)]):.2f} ms")
    print(f"D2H only: {wall(lambda: [h.copy_(d, non_blocking=True) for h, d in zip(hs, ds)]):.2f} ms")
    # both directions at once (the floor of an all-outputs step): H2D on one stream, D2H on another
    ho = [torch.empty(m, dtype=dt, pin_memory=True) for _ in range(tp)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            for h, d in zip(hs, ds):
                d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            for h, d in zip(ho, ds):
                h.copy_(d, non_blocking=True)
    print(f"H2D + D2H concurrently: {wall(both):.2f} ms")
    for mib in (4, 8, 12, 16, 24, 32):
        comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, mib << 20)
        comm.all_reduce_host(hs, fcfg)
        t_all = wall(lambda: comm.all_reduce_host(hs, fcfg))
        t_one = wall(lambda: comm.all_reduce_host(hs, fcfg, read_back=[r == 0 for r in range(tp)]))
        t_none = wall(lambda: comm.all_reduce_host(hs, fcfg, read_back=[False] * tp))
        print(f"chunk {mib:5d} MiB/rank: all outputs {t_all:7.2f} ms  rank-0 output {t_one:7.2f} ms  "
              f"no readback {t_none:7.2f} ms", flush=True)
    comm.close()


if __name__ == "__main__":
    main()
