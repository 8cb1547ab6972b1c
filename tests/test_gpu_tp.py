"""Caller integration: the flash all-reduce as the reduction
of a row-parallel linear layer, through the `torch.ops.flashcomm.all_reduce_`
custom op, eager and captured in a CUDA graph (the per-call epoch flags live in
device memory, so graph replays stay synchronised). Two processes share
cuda:0 over real CUDA IPC; results are bit-exact against the oracle."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, mode):
    import sys

    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        from oracle import flash_oracle as orc
        from paper_2412_04964_b200 import _lib, tp
        from paper_2412_04964_b200.comm import FlashComm

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        comm = FlashComm.from_process_group(device=0, slot_bytes=4 << 20)
        comm.set_timeout(30.0)
        comm.set_option(_lib.OPT_FUSED, 1 if mode == "fused" else 0)
        tp.set_comm(comm)
        tokens, hid, out = 64, 256, 1024
        layers = []
        for r in range(world):  # every rank can recompute every shard (deterministic seeds)
            torch.manual_seed(100 + r)
            layers.append(tp.FlashRowParallelLinear(hid // world, out, bits=4, device="cuda"))
        layer = layers[rank]

        def want(xs):
            parts = [(xs[r] @ layers[r].weight.t()).float().cpu().numpy().ravel() for r in range(world)]
            return orc.flash_all_reduce(parts, orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]

        def shards(seed):
            g = torch.Generator(device="cuda").manual_seed(seed)
            x = torch.randn(tokens, hid, device="cuda", generator=g).to(torch.bfloat16)
            return [x[:, r * hid // world:(r + 1) * hid // world].contiguous() for r in range(world)]

        with torch.no_grad():
            # eager
            xs = shards(1)
            y = layer(xs[rank])
            torch.cuda.synchronize()
            comm.check()
            ref = torch.from_numpy(want(xs)).to(torch.bfloat16).reshape(tokens, out)
            assert torch.equal(y.cpu().view(torch.int16), ref.view(torch.int16)), "eager"
            # CUDA graph: capture once, replay with new inputs
            static_x = xs[rank].clone()
            layer(static_x)  # warm (smem attributes, allocator)
            torch.cuda.synchronize()
            dist.barrier()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                static_y = layer(static_x)
            dist.barrier()
            for it in range(3):
                xs = shards(10 + it)
                static_x.copy_(xs[rank])
                graph.replay()
                torch.cuda.synchronize()
                comm.check()
                ref = torch.from_numpy(want(xs)).to(torch.bfloat16).reshape(tokens, out)
                assert torch.equal(static_y.cpu().view(torch.int16), ref.view(torch.int16)), f"replay {it}"
        dist.barrier()
        tp.clear_comms()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()[-1200:]))


@pytest.mark.parametrize("mode", ["fused", "split"])
def test_row_parallel_linear_eager_and_graph(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=300)
            res[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert res == {r: "ok" for r in range(world)}, res
