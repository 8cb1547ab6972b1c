"""Host-buffer flash all-reduce (fc_flash_all_reduce_host): the reference's own
call shape -- host arrays in, new host arrays out -- with the H2D copy, the
per-chunk all-reduce and the D2H copy pipelined on the communicator's streams.
Chunking must not change a single bit: every chunk run quantizes the same
groups as one whole-tensor call (spans are multiples of the plan unit), so the
host path is compared bitwise with the device-buffer path and with the
reference's golden outputs."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import flash_oracle as orc
from tests import golden_io as gio

pytestmark = pytest.mark.gpu

fc = pytest.importorskip("paper_2412_04964_b200")
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402


def _bits(t):
    return np.ascontiguousarray(t.float().numpy() if isinstance(t, torch.Tensor) else t).view(np.uint32)


def _case(n, m, dtype, seed, pinned=True):
    g = torch.Generator().manual_seed(seed)
    ts = [(torch.randn(m, generator=g) * (1 + r)).to(dtype) for r in range(n)]
    return [t.pin_memory() for t in ts] if pinned else ts


CASES = [
    # n, m, dtype, config, host chunk bytes (small -> many chunks)
    (4, 4 * 8192 * 6, torch.bfloat16, fc.FlashConfig.from_bits(4), 64 << 10),
    (8, 8 * 8192 * 5 + 4096, torch.bfloat16, fc.FlashConfig.from_bits(4), 96 << 10),  # ragged tail segment
    (4, 4 * 8192 * 4 - 100, torch.float16, fc.FlashConfig.from_bits(8), 32 << 10),  # last segment short
    (2, 2 * 8192 * 3, torch.float32, fc.FlashConfig.int6(), 16 << 10),
    (3, 3 * 96 * 200 + 17, torch.bfloat16, fc.FlashConfig.uniform(fc.CodecConfig(bits=4, group_size=96)), 8 << 10),
    (4, 4 * 8192 * 3, torch.bfloat16, fc.FlashConfig(fc.CodecConfig(bits=4), fc.PASSTHROUGH_FP16), 32 << 10),
    (8, 8 * 8192 * 2, torch.bfloat16, fc.FlashConfig.from_bits(8), 0),  # auto chunking
]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_host_pipeline_equals_device_call(i):
    n, m, dt, cfg, chunk = CASES[i]
    seg = -(-m // n)
    comm = FlashComm.local([0] * n, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, chunk)
    hs = _case(n, m, dt, seed=i)
    for odt in (dt, torch.float32):
        host = fc.flash_all_reduce(hs, cfg, comm=comm, out_dtype=odt).outputs
        dev = fc.flash_all_reduce([h.cuda() for h in hs], cfg, comm=comm, out_dtype=odt).outputs
        for r in range(n):
            assert not host[r].is_cuda and host[r].dtype == odt and host[r].shape == hs[r].shape
            assert torch.equal(host[r].view(torch.uint8), dev[r].cpu().view(torch.uint8)), (i, r, odt)
    comm.close()


def test_host_pipeline_golden_numpy():
    # numpy arrays in -> float32 host tensors out, equal to the reference's golden outputs
    for i in range(len(gio.flash_meta())):
        meta, xs, ref_out, _ = gio.flash_case(i)
        if meta["stage1"] == "fp16" and meta["stage2"] == "fp16":
            continue
        st = [fc.PASSTHROUGH_FP16 if s == "fp16" else fc.CodecConfig(bits=s[0], group_size=s[1], symmetric=s[2],
                                                                     rounding=s[3])
              for s in (meta["stage1"], meta["stage2"])]
        cfg = fc.FlashConfig(st[0], st[1], chunk_size=meta["chunk"])
        run = fc.flash_all_reduce(list(xs), cfg)
        for o in run.outputs:
            assert not o.is_cuda
            assert np.array_equal(_bits(o.numpy()), _bits(ref_out)), i
        assert run.wire_bytes_per_rank == meta["wire_bytes_per_rank"]


def test_host_pipeline_oracle_pageable_and_partial_readback():
    n, m = 4, 4 * 8192 * 2 + 300
    hs = _case(n, m, torch.float32, seed=7, pinned=False)
    cfg = fc.FlashConfig.from_bits(4)
    ref = orc.flash_all_reduce([h.numpy() for h in hs], orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
    run = fc.flash_all_reduce(hs, cfg)
    for o in run.outputs:
        assert np.array_equal(_bits(o.numpy()), _bits(ref))
    comm = FlashComm.local([0] * n, slot_bytes_for(-(-m // n), cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, 32 << 10)
    outs = comm.all_reduce_host(hs, cfg, read_back=[False, True, False, False])
    assert outs[0] is None and outs[2] is None and outs[3] is None
    assert np.array_equal(_bits(outs[1].numpy()), _bits(ref))
    # caller-supplied (reused) host outputs through the public call
    mine = [torch.full((m,), 7.0).pin_memory(), None, torch.empty(m), None]
    run = fc.flash_all_reduce(hs, cfg, comm=comm, outs=mine)
    assert run.outputs[0].data_ptr() == mine[0].data_ptr() and run.outputs[1] is None
    assert np.array_equal(_bits(mine[0].numpy()), _bits(ref)) and np.array_equal(_bits(mine[2].numpy()), _bits(ref))
    with pytest.raises(fc.DomainError):
        fc.flash_all_reduce(hs, cfg, comm=comm, outs=[torch.empty(m - 1)] * n)
    comm.close()


def test_host_pipeline_errors_and_recovery():
    n, m = 4, 4 * 8192
    cfg = fc.FlashConfig.from_bits(4)
    hs = _case(n, m, torch.float32, seed=3)
    comm = FlashComm.local([0] * n, slot_bytes_for(m // n, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, 16 << 10)
    hs[1][5000] = float("nan")
    with pytest.raises(fc.DomainError):
        fc.flash_all_reduce(hs, cfg, comm=comm)
    hs[1][5000] = 0.0
    ref = orc.flash_all_reduce([h.numpy() for h in hs], orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
    run = fc.flash_all_reduce(hs, cfg, comm=comm)
    assert np.array_equal(_bits(run.outputs[2].numpy()), _bits(ref))
    with pytest.raises(fc.ProtocolError):
        fc.flash_all_reduce([torch.zeros(8), torch.zeros(9)], cfg)
    with pytest.raises(fc.DomainError):
        fc.flash_all_reduce([torch.zeros(0)] * 2, cfg)
    with pytest.raises(fc.ConfigError):
        fc.flash_all_reduce([torch.zeros(1024)] * 4, fc.FlashConfig.from_bits(4, chunk_size=128))
    with pytest.raises(fc.ConfigError):  # bf16 in, fp16 out has no kernel
        comm.all_reduce_host([h.to(torch.bfloat16) for h in hs], cfg, out_dtype=torch.float16)
    x = torch.arange(10, dtype=torch.float32)
    one = fc.flash_all_reduce([x], cfg)
    assert torch.equal(one.outputs[0], x) and not one.outputs[0].is_cuda
    comm.close()


def _ipc_host_worker(rank, world, port, q):
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        n, m = world, world * 8192 * 5 + 1000  # ragged tail segment
        cfg = fc.FlashConfig.from_bits(4)
        comm = FlashComm.from_process_group(device=0, slot_bytes=slot_bytes_for(-(-m // n), cfg.stage1_codec,
                                                                               cfg.stage2_codec))
        comm.set_timeout(30.0)
        comm.set_option(_lib.OPT_HOST_CHUNK_BYTES, 48 << 10)  # many chunks, same on every rank
        for variant in range(3):  # fresh inputs every call: a chunk run that read stale staging would show
            hs = _case(n, m, torch.bfloat16, seed=11 + variant)
            ref = orc.flash_all_reduce([h.float().numpy() for h in hs], orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
            got = comm.all_reduce_host_rank(hs[rank], cfg, out_dtype=torch.float32)
            bad = (got != torch.from_numpy(ref)).nonzero().ravel()
            assert bad.numel() == 0, (variant, bad.numel(), bad[:4].tolist(), m)
        for odt in (torch.bfloat16, torch.float32):
            want = torch.from_numpy(ref).to(odt)
            for order in range(3):  # host, device, host: no state leaks between the two forms
                if order == 1:
                    got = comm.all_reduce(hs[rank].cuda(), cfg, out_dtype=odt, check=True).cpu()
                else:
                    got = comm.all_reduce_host_rank(hs[rank], cfg, out_dtype=odt)
                    assert not got.is_cuda
                bad = (got.float() != want.float()).nonzero().ravel()
                assert bad.numel() == 0, (odt, order, bad.numel(), bad[:4].tolist(), bad[-4:].tolist(), m)
        dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()[-1200:]))


def test_host_pipeline_ipc_ranks():
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_host_worker, args=(r, world, port, q)) for r in range(world)]
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
