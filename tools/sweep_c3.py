"""C3 (BASELINE.json configs[2]): INT8 vs INT4 message-size sweep, 64 KB to
512 MB of bf16 per rank, at TP = 2 / 4 / 8, every TP rank emulated as a
logical rank of one B200 (the only GPU this build has). Each point is device
time from a CUDA graph of back-to-back all-reduces (host launch path excluded),
reported as latency, algbw (nccl-tests convention e*M/t), whole-job GB/s and
the fraction of the emulated HBM roofline (all ranks' algorithmic bytes).

usage: python tools/sweep_c3.py [--max-mb 512] [--out gpurun_out/sweep_c3.jsonl]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_04964_b200 as fc  # noqa: E402
from bench import graph_time, load_peaks  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=512)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep_c3.jsonl"))
    args = ap.parse_args()
    peak = load_peaks()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    e = 2
    rows = []
    with open(args.out, "w") as fh:
        for tp in (2, 4, 8):
            nbytes = 64 << 10
            while nbytes <= args.max_mb << 20:
                m = nbytes // e
                seg = -(-m // tp)
                for bits in (8, 4):
                    cfg = fc.FlashConfig.from_bits(bits)
                    comm = FlashComm.local([0] * tp, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
                    ins = [torch.randn(m, device=dev).to(torch.bfloat16) for _ in range(tp)]
                    outs = [torch.empty_like(t) for t in ins]
                    reps = 20 if nbytes <= (8 << 20) else 5
                    ms = graph_time(lambda: comm.all_reduce_local(ins, cfg, outs=outs, check=False), reps, stream)
                    comm.check()
                    w = cfg.stage1_codec.wire_byte_len(seg) + cfg.stage2_codec.wire_byte_len(seg)
                    alg = tp * (2 * e * m + 2 * (tp - 1) * w)
                    row = {"config": "C3", "tp": tp, "bits": bits, "bytes_per_rank": nbytes, "latency_us": ms * 1e3,
                           "algbw_gbs": e * m / (ms * 1e-3) / 1e9, "job_gbs": tp * e * m / (ms * 1e-3) / 1e9,
                           "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak["hbm_gbs"], "nvlink_bytes_per_rank": (tp - 1) * w,
                           "emulated": f"{tp} logical ranks on 1 GPU", "peak": peak}
                    fh.write(json.dumps(row) + "\n")
                    fh.flush()
                    rows.append(row)
                    comm.close()
                    del ins, outs
                nbytes *= 2
            torch.cuda.empty_cache()
    for r in rows:
        print(f"tp={r['tp']} int{r['bits']} {r['bytes_per_rank'] >> 10:8d} KiB  {r['latency_us']:9.1f} us  "
              f"algbw {r['algbw_gbs']:7.1f} GB/s  hbm {r['hbm_frac'] * 100:5.1f}%")


if __name__ == "__main__":
    main()
