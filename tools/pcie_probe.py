"""Host<->device copy probe for the end-to-end (host-buffer) path: pinned H2D and
D2H bandwidth, alone and concurrently (PCIe duplex), whole-tensor vs chunked
and strided (cudaMemcpy2DAsync-shaped) copies.

usage: python tools/pcie_probe.py [--mb 128] [--ranks 8]
"""

from __future__ import annotations

import argparse
import time

import torch


def timed(fn, reps=3):
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=128)
    ap.add_argument("--ranks", type=int, default=8)
    args = ap.parse_args()
    n = args.mb << 20
    R = args.ranks
    hs = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(R)]
    ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(R)]
    ho = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(R)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    tot = R * n

    def h2d():
        with torch.cuda.stream(s1):
            for h, d in zip(hs, ds):
                d.copy_(h, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            for h, d in zip(ho, ds):
                h.copy_(d, non_blocking=True)

    def both():
        h2d()
        d2h()

    def h2d_chunked(k=16):
        c = n // k
        with torch.cuda.stream(s1):
            for i in range(k):
                for h, d in zip(hs, ds):
                    d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)

    t = timed(h2d)
    print(f"H2D {R}x{args.mb} MiB: {t * 1e3:.2f} ms  {tot / t / 1e9:.1f} GB/s")
    t = timed(d2h)
    print(f"D2H {R}x{args.mb} MiB: {t * 1e3:.2f} ms  {tot / t / 1e9:.1f} GB/s")
    t = timed(both)
    print(f"H2D+D2H concurrent: {t * 1e3:.2f} ms  {2 * tot / t / 1e9:.1f} GB/s both directions")
    for k in (8, 32, 128):
        t = timed(lambda: h2d_chunked(k))
        print(f"H2D chunked x{k} ({n // k >> 10} KiB copies): {t * 1e3:.2f} ms  {tot / t / 1e9:.1f} GB/s")
    # pageable source for comparison
    pg = [torch.empty(n, dtype=torch.uint8) for _ in range(2)]
    t = timed(lambda: [d.copy_(h) for h, d in zip(pg, ds)])
    print(f"H2D pageable 2x{args.mb} MiB: {t * 1e3:.2f} ms  {2 * n / t / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
