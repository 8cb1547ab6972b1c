"""One process per rank over CUDA IPC (the torchrun path), exercised on a
single GPU: 2-8 processes share cuda:0, map each other's blocks with
cudaIpcOpenMemHandle and run the fused flag-synchronised kernel (OPT_FUSED 1)
or the phase-split kernels with IPC barriers (OPT_FUSED 0, OPT_ONESHOT 0), or the
one-launch small-message kernel (default at decode sizes, k_small). Parity vs the
oracle, plus the fault path: a rank that never arrives -> ProtocolError
naming the stuck peer (fabric.py:158-178)."""

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

        import paper_2412_04964_b200 as fc
        from oracle import flash_oracle as orc
        from paper_2412_04964_b200 import _lib
        from paper_2412_04964_b200.comm import FlashComm

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        comm = FlashComm.from_process_group(device=0, slot_bytes=1 << 20)
        comm.set_timeout(20.0)
        if mode == "fused":
            comm.set_option(_lib.OPT_FUSED, 1)
        if mode in ("split", "mfsplit"):
            comm.set_option(_lib.OPT_FUSED, 0)
            comm.set_option(_lib.OPT_ONESHOT, 0)
        if mode == "generic":
            comm.set_option(_lib.OPT_FAST, 0)
        # 3 tiles per segment: the default ("small") takes the one-launch small-message kernel
        # (k_small); "split" / "fused" force the streaming kernels at the same size
        m = 8192 * world * 3 + (0 if mode != "generic" else 100)
        xs = orc.gen_rank_activations(8192, -(-m // 8192), 21, world)
        xs = [orc.round_to_bf16(x.ravel()[:m]) for x in xs]
        if mode in ("minifloat", "mfstream", "mfsplit"):
            # e4m3 stages: float32 outputs take the lane-8 kernels with IPC barriers, bf16 outputs
            # the fused streaming kernel on MfSpec (flag-synchronised across the processes), or
            # ("mfsplit") the three streaming phase kernels with IPC barriers
            cfg = fc.FlashConfig.uniform(fc.CodecConfig(number_format="e4m3"))
            oc = orc.Codec(kind="e4m3")
        else:
            cfg = fc.FlashConfig.from_bits(4)
            oc = orc.Codec(bits=4)
        want = orc.flash_all_reduce(xs, oc, oc).outputs[0]
        for it in range(3):
            x = torch.from_numpy(xs[rank]).cuda().to(torch.bfloat16)
            if mode in ("mfstream", "mfsplit"):
                out = comm.all_reduce(x, cfg, out_dtype=torch.bfloat16, check=True)
                launches = comm.get_option(_lib.OPT_LAST_LAUNCHES)
                assert launches == (2 if mode == "mfstream" else 6), launches  # fused / split + 2 barriers
                got = out.view(torch.int16).cpu().numpy()
                assert np.array_equal(got, orc.f32_to_bf16_bits(want).view(np.int16)), f"iteration {it}"
                continue
            out = comm.all_reduce(x, cfg, out_dtype=torch.float32, check=True)
            if mode == "fused":  # the fused kernel itself ran (fp32 outputs): epoch bump + k_fstream
                assert comm.get_option(_lib.OPT_LAST_LAUNCHES) == 2, comm.get_option(_lib.OPT_LAST_LAUNCHES)
            got = out.cpu().numpy()
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"iteration {it}"
        dist.barrier()
        comm.teardown_check()  # every rank ran the same rounds
        if mode == "timeout":
            if rank == 0:
                comm.set_timeout(2.0)
                x = torch.from_numpy(xs[0]).cuda().to(torch.bfloat16)
                comm.all_reduce(x, cfg)
                try:
                    comm.check()
                    raise AssertionError("expected ProtocolError")
                except fc.ProtocolError as e:
                    assert "timed out waiting on rank" in str(e), str(e)
            dist.barrier()
            # rank 0 ran a round rank 1 never joined: unconsumed at teardown (fabric.py:228-236)
            try:
                comm.teardown_check()
                raise AssertionError("expected ProtocolError")
            except fc.ProtocolError as e:
                assert "unconsumed" in str(e), str(e)
        if mode == "unaligned":
            # a view 2 bytes into its storage: refused before any launch (the kernel path every
            # rank must share depends on alignment), so no rank waits on a peer
            base = torch.zeros(8 * 8192 * world + 8, device="cuda", dtype=torch.bfloat16)
            try:
                comm.all_reduce(base[1:1 + 8 * 8192 * world], cfg)
                raise AssertionError("expected DomainError")
            except fc.DomainError as e:
                assert "aligned" in str(e), str(e)
            dist.barrier()
        if mode == "abort":
            # ranks 0 and 1 call, rank 2 never does; rank 0 (2 s timeout) gives up first and its
            # abort reaches rank 1 (60 s timeout) at once (fabric.py:168-172, 203-205)
            import time
            if rank < 2:
                comm.set_timeout(2.0 if rank == 0 else 60.0)
                x = torch.from_numpy(xs[rank]).cuda().to(torch.bfloat16)
                t0 = time.perf_counter()
                comm.all_reduce(x, cfg)
                try:
                    comm.check()
                    raise AssertionError("expected ProtocolError")
                except fc.ProtocolError as e:
                    assert "rank 0 timed out waiting on rank" in str(e), str(e)  # the originator
                assert time.perf_counter() - t0 < 20.0, "abort did not propagate"
            dist.barrier()
        comm.close()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, repr(e) + traceback.format_exc()[-800:]))


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=240)
            res[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert res == {r: "ok" for r in range(world)}, res


@pytest.mark.parametrize("world,mode", [(2, "fused"), (4, "fused"), (8, "fused"), (2, "split"), (4, "split"),
                                        (8, "split"), (2, "small"), (4, "small"), (8, "small"), (3, "generic"),
                                        (4, "minifloat"), (8, "mfstream"), (4, "mfsplit")])
def test_ipc_parity(world, mode):
    _run(world, mode)


def test_ipc_unaligned_buffer_refused():
    _run(2, "unaligned")


def test_ipc_timeout_names_peer():
    _run(2, "timeout")


def test_ipc_abort_propagates():
    _run(3, "abort")
