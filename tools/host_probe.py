"""Host launch overhead probe: the same all-reduce timed eagerly (CUDA events,
host launch path included) and replayed from a CUDA graph (device time only),
plus the host wall time per call, for the bench configurations.

usage: python tools/host_probe.py [--configs c1,c2,c4] [--reps 50]
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
from bench import CONFIGS, _dtype, _events_time, graph_time  # noqa: E402
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c4")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for name in args.configs.split(","):
        cfg = CONFIGS[name]
        tp, dt, m = cfg["tp"], _dtype(cfg["dtype"]), math.prod(cfg["shape"])
        seg = -(-m // tp)
        fcfg = fc.FlashConfig.from_bits(cfg["bits"], group_size=cfg["group"])
        comm = FlashComm.local([0] * tp, slot_bytes_for(seg, fcfg.stage1_codec, fcfg.stage2_codec))
        ins = [torch.randn(m, device=dev).to(dt) for _ in range(tp)]
        outs = [torch.empty_like(t) for t in ins]
        step = lambda: comm.all_reduce_local(ins, fcfg, outs=outs, check=False)  # noqa: E731
        for _ in range(5):
            step()
        torch.cuda.synchronize()
        eager, _ = _events_time(step, args.reps, stream)
        graph = graph_time(step, args.reps, stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            step()
        host = (time.perf_counter() - t0) / args.reps
        torch.cuda.synchronize()
        # the C-ABI call alone (ctypes arguments prebuilt) and a trivial C-ABI call
        import ctypes as C
        from paper_2412_04964_b200.codec import fc_dtype
        N = tp
        pin = (C.c_void_p * N)(*[t.data_ptr() for t in ins])
        pout = (C.c_void_p * N)(*[o.data_ptr() for o in outs])
        pst = (C.c_void_p * N)(*[stream.cuda_stream] * N)
        cc = comm._cfg(fcfg)
        fn, h, d = _lib.lib().fc_flash_all_reduce_local, comm._h, fc_dtype(dt)
        t0 = time.perf_counter()
        for _ in range(args.reps):
            fn(h, pin, pout, m, d, d, C.byref(cc), pst)
        raw = (time.perf_counter() - t0) / args.reps
        torch.cuda.synchronize()
        per_phase = {}
        for ph in (1, 2, 4):
            comm.set_option(_lib.OPT_FUSED, 0)
            comm.set_option(_lib.OPT_PHASES, ph)
            fn(h, pin, pout, m, d, d, C.byref(cc), pst)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.reps):
                fn(h, pin, pout, m, d, d, C.byref(cc), pst)
            per_phase[ph] = (time.perf_counter() - t0) / args.reps * 1e6
            torch.cuda.synchronize()
        comm.set_option(_lib.OPT_PHASES, 0)
        comm.set_option(_lib.OPT_FUSED, -1)
        print(f"{name}: raw C call per phase (us): " + "  ".join(f"{k}:{v:.1f}" for k, v in per_phase.items()))
        x = torch.empty(16, device=dev)
        t0 = time.perf_counter()
        for _ in range(args.reps):
            x.zero_()
        print(f"{name}: torch zero_ launch {(time.perf_counter() - t0) / args.reps * 1e6:.1f} us", flush=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            comm._cfg(fcfg)
        cfgt = (time.perf_counter() - t0) / args.reps
        t0 = time.perf_counter()
        for _ in range(args.reps):
            comm.get_option(_lib.OPT_LAST_LAUNCHES)
        triv = (time.perf_counter() - t0) / args.reps
        print(f"{name}: raw C call {raw * 1e6:7.1f} us  _cfg {cfgt * 1e6:6.1f} us  trivial C call {triv * 1e6:6.1f} us",
              flush=True)
        launches = comm.get_option(_lib.OPT_LAST_LAUNCHES)
        print(f"{name}: eager {eager * 1e3:8.1f} us  graph {graph * 1e3:8.1f} us  host/call {host * 1e6:7.1f} us  "
              f"launches {launches}", flush=True)
        comm.close()


if __name__ == "__main__":
    main()
