"""Multi-process host logic of the one-rank-per-GPU path, on CPU (gloo,
world_size 2 and 3): IPC-handle exchange in rank order, and the per-rank
segment protocol (each rank owns segment r; stage-1 pieces go to their
owner, stage-2 payloads to everyone) agreeing with the list-form oracle.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import flash_oracle as orc
    from paper_2412_04964_b200.comm import exchange_handles

    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        # 1) handle exchange
        mine = bytes([rank] * 64)
        allh = exchange_handles(mine)
        assert allh == b"".join(bytes([r] * 64) for r in range(world))
        # 2) per-rank protocol over the wire (bytes), vs the list-form oracle
        m = 5000 * world + 3
        xs = orc.gen_rank_activations(1000, -(-m // 1000), 5, world)
        xs = [x.ravel()[:m] for x in xs]
        c1, c2 = orc.Codec(bits=4, group_size=64), orc.Codec(bits=8, group_size=64)
        seg = -(-m // world)
        pad = np.zeros(world * seg, np.float32)
        pad[:m] = xs[rank]
        sent = [orc.quantize(pad[j * seg:(j + 1) * seg], c1) for j in range(world)]
        got = [None] * world
        dist.all_gather_object(got, [s.wire_bytes() for s in sent])
        parts = []
        for s in range(world):
            blob = got[s][rank]
            ref = orc.quantize(np.zeros(seg, np.float32), c1)  # shape donor
            codes = orc.unpack(np.frombuffer(blob[: (seg + 1) // 2], np.uint8), seg, 4)
            g = -(-seg // 64)
            sc = np.frombuffer(blob[(seg + 1) // 2:(seg + 1) // 2 + 2 * g], np.float16)
            zs = np.frombuffer(blob[(seg + 1) // 2 + 2 * g:], np.uint8)
            parts.append(orc.dequantize(orc.QSeg(codes, sc, zs, seg, c1)))
            del ref
        red = orc.sequential_sum(parts)
        q2 = orc.quantize(red, c2)
        st2 = [None] * world
        dist.all_gather_object(st2, q2.wire_bytes())
        out = []
        for j in range(world):
            blob = st2[j]
            g = -(-seg // 64)
            out.append(orc.dequantize(orc.QSeg(np.frombuffer(blob[:seg], np.uint8).copy(),
                                               np.frombuffer(blob[seg:seg + 2 * g], np.float16),
                                               np.frombuffer(blob[seg + 2 * g:], np.uint8), seg, c2)))
        mine_out = np.concatenate(out)[:m]
        want = orc.flash_all_reduce(xs, c1, c2).outputs[0]
        assert np.array_equal(mine_out.view(np.uint32), want.view(np.uint32))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_multirank_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}
