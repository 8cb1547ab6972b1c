"""Stress the per-rank host-buffer pipeline over CUDA IPC (2 processes, one GPU):
many chunked calls, bitwise against the oracle, under an FC_OPT_STREAM_MASK value.
usage: python tools/ipc_host_stress.py <mask> <iterations> [host|device]"""
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, q, mask, iters, form):
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        import paper_2412_04964_b200 as fc
        from oracle import flash_oracle as orc
        from paper_2412_04964_b200 import _lib
        from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        n, m = world, world * 8192 * 5 + 1000
        cfg = fc.FlashConfig.from_bits(4)
        comm = FlashComm.from_process_group(device=0, slot_bytes=slot_bytes_for(-(-m // n), cfg.stage1_codec,
                                                                                 cfg.stage2_codec))
        comm.set_timeout(30.0)
        comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, int(os.environ.get("CHUNK", 48 << 10)))
        comm.set_option(_lib.OPT_STREAM_MASK, mask)
        g = torch.Generator().manual_seed(11)
        hs = [(torch.randn(m, generator=g) * (1 + r)).to(torch.bfloat16).pin_memory() for r in range(n)]
        ref = orc.flash_all_reduce([h.float().numpy() for h in hs], orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
        want = torch.from_numpy(ref).to(torch.bfloat16)
        hs_b = [(h.float() * -0.5).to(torch.bfloat16).pin_memory() for h in hs]
        ref_b = orc.flash_all_reduce([h.float().numpy() for h in hs_b], orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
        want_b = torch.from_numpy(ref_b).to(torch.bfloat16)
        bad_calls = []
        for it in range(iters):
            if it % 2:  # alternate two inputs so a run that read stale staging cannot pass
                hs_it, want_it = hs_b, want_b
            else:
                hs_it, want_it = hs, want
            if form == "host":
                got = comm.all_reduce_host_rank(hs_it[rank], cfg)
            else:
                got = comm.all_reduce(hs_it[rank].cuda(), cfg, check=True).cpu()
            bad = (got.float() != want_it.float()).nonzero().ravel()
            if bad.numel():
                bad_calls.append((it, bad.numel(), int(bad[0]), int(bad[-1])))
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, bad_calls))
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()[-800:]))


if __name__ == "__main__":
    mask, iters = int(sys.argv[1]), int(sys.argv[2])
    form = sys.argv[3] if len(sys.argv) > 3 else "host"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, mask, iters, form)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
    print(f"mask {mask} {form}: {res}", flush=True)
