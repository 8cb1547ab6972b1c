"""GPU parity of the flash all-reduce (libflashcomm sm_100a kernels) against
the reference's golden outputs, its own wire messages (through the oracle's
per-slot restatement) and its reported error numbers.

Several logical ranks share cuda:0 (the reference's list-of-tensors call);
the same kernels serve one rank per GPU. Float32 outputs must equal the
reference bit for bit; bf16/fp16 outputs equal its RNE rounding.
"""

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

MODES = {"fused": dict(fused=1, fast=1), "split": dict(fused=0, fast=1), "generic": dict(fused=1, fast=0)}


def _stage(spec):
    if spec == "fp16":
        return fc.PASSTHROUGH_FP16
    bits, g, sym, rnd = spec
    return fc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)


def _comm(n, seg, cfg, mode, slot_bytes=None):
    comm = FlashComm.local([0] * n, slot_bytes or slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, MODES[mode]["fused"])
    comm.set_option(_lib.OPT_FAST, MODES[mode]["fast"])
    return comm


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("i", range(len(gio.flash_meta())))
def test_flash_golden(i, mode):
    meta, xs, ref_out, ref_exact = gio.flash_case(i)
    n, m = meta["n"], meta["m"]
    cfg = fc.FlashConfig(_stage(meta["stage1"]), _stage(meta["stage2"]), chunk_size=meta["chunk"])
    seg = -(-m // n)
    comm = _comm(n, seg, cfg, mode)
    ts = [torch.from_numpy(x).cuda() for x in xs]
    run = fc.flash_all_reduce(ts, cfg, comm=comm)
    for o in run.outputs:
        assert np.array_equal(_bits(o.cpu().numpy()), _bits(ref_out))
    assert run.wire_bytes_per_rank == meta["wire_bytes_per_rank"]
    assert run.qdq_passes == meta["qdq"] and run.reduce_elems_per_rank == meta["reduce_elems"]
    # stage buffers: the reference's per-piece wire messages restated per slot
    s1, s2 = gio.oracle_stage(meta["stage1"]), gio.oracle_stage(meta["stage2"])
    res = orc.flash_all_reduce(xs, s1, s2, meta["chunk"])
    for j in range(n):
        for s in range(n):
            if s != j:
                got = comm.slot(j, 1, s, cfg.stage1_codec).to_bytes()
                assert got == res.stage1[j][s].wire_bytes(), f"stage-1 slot {j}<-{s}"
        p = (j + 1) % n
        assert comm.slot(p, 2, j, cfg.stage2_codec).to_bytes() == res.stage2[j].wire_bytes(), f"stage-2 {j}"
    comm.close()


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_half_in_half_out(n, dtype):
    m = 4 * 8192 * n + 136
    xs = orc.gen_rank_activations(8192, -(-m // 8192), 11, n)
    xs = [x.ravel()[:m] for x in xs]
    ts = [torch.from_numpy(x).cuda().to(dtype) for x in xs]
    xr = [t.float().cpu().numpy() for t in ts]
    cfg = fc.FlashConfig.from_bits(4)
    run = fc.flash_all_reduce(ts, cfg)
    ref = orc.flash_all_reduce(xr, orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
    want = torch.from_numpy(ref).to(dtype)
    for o in run.outputs:
        assert o.dtype == dtype
        assert torch.equal(o.cpu().view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("mode", ["fused", "split", "generic"])
def test_many_rounds_transparent(mode):
    # slots far smaller than a segment: the call runs in rounds; results unchanged
    n, m = 4, 4 * 8192 * 9 + 4 * 1000
    rng = np.random.default_rng(3)
    xs = [orc.round_to_bf16((rng.standard_normal(m) * 2).astype(np.float32)) for _ in range(n)]
    cfg = fc.FlashConfig.int6()
    comm = _comm(n, 0, cfg, mode, slot_bytes=3 * 8192 + 4096)
    ts = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in xs]
    run = fc.flash_all_reduce(ts, cfg, comm=comm, out_dtype=torch.float32)
    ref = orc.flash_all_reduce(xs, orc.Codec(bits=4), orc.Codec(bits=8)).outputs[0]
    for o in run.outputs:
        assert np.array_equal(_bits(o.cpu().numpy()), _bits(ref))
    comm.close()


def test_in_place_and_back_to_back():
    n, m = 8, 8 * 8192 * 3
    cfg = fc.FlashConfig.from_bits(4)
    comm = _comm(n, m // n, cfg, "fused")
    for it in range(5):
        g = torch.Generator(device="cuda").manual_seed(it)
        ts = [torch.randn(m, device="cuda", generator=g).to(torch.bfloat16) for _ in range(n)]
        xr = [t.float().cpu().numpy() for t in ts]
        ref = orc.flash_all_reduce(xr, orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
        outs = comm.all_reduce_local(ts, cfg, outs=ts)  # in place
        want = torch.from_numpy(ref).to(torch.bfloat16)
        for o in outs:
            assert torch.equal(o.cpu().view(torch.int16), want.view(torch.int16))
    comm.close()


def test_decode_sizes_tp8():
    # C4: bs x 8192 bf16 at TP=8 (1 to 8 tiles per segment)
    cfg = fc.FlashConfig.from_bits(4)
    for bs in (8, 16, 32, 64):
        m = bs * 8192
        g = torch.Generator(device="cuda").manual_seed(bs)
        ts = [torch.randn(m, device="cuda", generator=g).to(torch.bfloat16) for _ in range(8)]
        xr = [t.float().cpu().numpy() for t in ts]
        ref = orc.flash_all_reduce(xr, orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
        run = fc.flash_all_reduce(ts, cfg, out_dtype=torch.float32)
        assert np.array_equal(_bits(run.outputs[3].cpu().numpy()), _bits(ref))


def test_nonfinite_raises_and_comm_recovers():
    n, m = 4, 4 * 8192
    cfg = fc.FlashConfig.from_bits(4)
    comm = _comm(n, m // n, cfg, "fused")
    ts = [torch.randn(m, device="cuda") for _ in range(n)]
    ts[2][777] = float("inf")
    with pytest.raises(fc.DomainError):
        fc.flash_all_reduce(ts, cfg, comm=comm)
    ts[2][777] = 0.0
    xr = [t.cpu().numpy() for t in ts]
    run = fc.flash_all_reduce(ts, cfg, comm=comm)
    ref = orc.flash_all_reduce(xr, orc.Codec(bits=4), orc.Codec(bits=4)).outputs[0]
    assert np.array_equal(_bits(run.outputs[0].cpu().numpy()), _bits(ref))
    comm.close()


def test_api_errors():
    cfg = fc.FlashConfig.from_bits(4, group_size=128, chunk_size=128)
    with pytest.raises(fc.ConfigError):  # test_collectives.py:176-179
        fc.flash_all_reduce([torch.zeros(1024, device="cuda")] * 4, cfg)
    with pytest.raises(fc.ProtocolError):
        fc.flash_all_reduce([torch.zeros(4, device="cuda"), torch.zeros(5, device="cuda")], fc.FlashConfig.from_bits(4))
    with pytest.raises(fc.DomainError):
        fc.flash_all_reduce([torch.zeros(0, device="cuda")] * 2, fc.FlashConfig.from_bits(4))
    with pytest.raises(fc.ConfigError):
        fc.run_collective("flash", [torch.zeros(8, device="cuda")] * 2)
    with pytest.raises(fc.ConfigError):
        fc.flash_all_reduce([torch.zeros(8, device="cuda")] * 2, fc.FlashConfig.from_bits(4),
                            topology=fc.FabricTopology(world_size=3))
    x = torch.arange(10, dtype=torch.float32, device="cuda")
    run = fc.flash_all_reduce([x], fc.FlashConfig.from_bits(4, group_size=2))
    assert torch.equal(run.outputs[0], x) and run.qdq_passes == 0


def test_exact_and_order():
    xs = [torch.tensor([1e8], device="cuda"), torch.tensor([-1e8], device="cuda"), torch.tensor([1.0], device="cuda")]
    assert float(fc.all_reduce_exact(xs).outputs[0][0]) == 1.0


def test_baseline_mse_table():
    # 1024x8192 outlier activations (bf16), flash vs exact fp32
    rep = gio.reports()["baseline_mse"]
    for n in (2, 4, 8):
        xs = orc.gen_rank_activations(8192, 1024, 0, n)
        ts = [torch.from_numpy(orc.round_to_bf16(x)).cuda().to(torch.bfloat16) for x in xs]
        exact = fc.all_reduce_exact(ts).outputs[0]
        for bits in (8, 6, 4):
            out = fc.flash_all_reduce(ts, fc.FlashConfig.from_bits(bits), out_dtype=torch.float32).outputs[0]
            got = fc.mse(out, exact)
            assert got == pytest.approx(rep[f"n{n}_b{bits}"], rel=1e-6), (n, bits)


def test_rs_vs_ag_reproduced():
    # workload.py:176-200 on the default profile (4096 x 16)
    rep = gio.reports()["rs_vs_ag"]
    for key, (half_ref, full_ref) in rep.items():
        n, bits = int(key.split("_")[0][1:]), int(key.split("_")[1][1:])
        xs = [torch.from_numpy(x).cuda() for x in orc.gen_rank_activations(4096, 16, 0, n)]
        exact = fc.all_reduce_exact(xs).outputs[0]
        half = fc.flash_all_reduce(xs, fc.FlashConfig(fc.CodecConfig(bits=bits), fc.PASSTHROUGH_FP16)).outputs[0]
        full_cfg = fc.FlashConfig.int6() if bits == 6 else fc.FlashConfig.from_bits(bits)
        full = fc.flash_all_reduce(xs, full_cfg).outputs[0]
        assert fc.mse(half, exact) == pytest.approx(half_ref, rel=1e-9)
        assert fc.mse(full, exact) == pytest.approx(full_ref, rel=1e-9)


@pytest.mark.slow
def test_c2_full_size_segment_spot_check():
    # C2: TP=8, INT4 g128, bf16 [8,1024,8192] per rank, all 8 ranks on one GPU.
    n, m = 8, 8 * 1024 * 8192
    g = torch.Generator(device="cuda").manual_seed(1234)
    ts = [torch.randn(m, device="cuda", generator=g).to(torch.bfloat16) for _ in range(n)]
    cfg = fc.FlashConfig.from_bits(4)
    run = fc.flash_all_reduce(ts, cfg)
    seg = m // n
    for r in range(1, n):  # every rank decodes the same stage-2 payloads
        assert torch.equal(run.outputs[r], run.outputs[0])
    j = 5  # segment j depends only on segment j of every rank
    xr = [t[j * seg:(j + 1) * seg].float().cpu().numpy() for t in ts]
    c = orc.Codec(bits=4)
    red = orc.sequential_sum([orc.dequantize(orc.quantize(x, c)) for x in xr])
    ref = orc.dequantize(orc.quantize(red, c))
    want = torch.from_numpy(ref).to(torch.bfloat16)
    assert torch.equal(run.outputs[0][j * seg:(j + 1) * seg].cpu().view(torch.int16), want.view(torch.int16))


@pytest.mark.parametrize("bits", [4, 8, 6])
def test_stream_kernels_match_generic_tp8(bits):
    """The bulk-copy streaming kernels (ring reuse over many tiles per CTA; the
    group-lane reduce's piece ring wraps many times) are bit-identical to the
    independent one-thread-per-group generic kernels (OPT_FAST 0) at TP=8,
    1024x8192 per rank, twice in a row (regression for shared-memory WAR races
    between consumer loads and the next tile's bulk copy). The oracle pins
    these sizes through tests/test_gpu_fullsize.py's reference digests."""
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    tp, M = 8, 1024 * 8192
    cfg = fc.FlashConfig.from_bits(bits)
    comm = FlashComm.local([0] * tp, slot_bytes_for(M // tp, cfg.stage1_codec, cfg.stage2_codec))
    try:
        comm.set_option(_lib.OPT_FUSED, 0)
        g = torch.Generator(device="cuda").manual_seed(bits)
        ins = [torch.randn(M, device="cuda", generator=g).to(torch.bfloat16) for _ in range(tp)]
        comm.set_option(_lib.OPT_FAST, 0)
        ref = [o.clone() for o in comm.all_reduce_local(ins, cfg, out_dtype=torch.bfloat16)]
        comm.set_option(_lib.OPT_FAST, 1)
        for fused in (0, 1):
            comm.set_option(_lib.OPT_FUSED, fused)
            for _ in range(2):
                outs = comm.all_reduce_local(ins, cfg, out_dtype=torch.bfloat16)
                for r in range(tp):
                    assert torch.equal(outs[r].view(torch.int16), ref[r].view(torch.int16)), (fused, r)
    finally:
        comm.close()


@pytest.mark.parametrize("mode", ["fused", "split"])
@pytest.mark.parametrize("bits,g,sym,rnd", [(4, 128, True, "nearest-even"), (8, 64, True, "nearest-even"),
                                            (4, 256, False, "ceil"), (8, 32, False, "ceil"),
                                            (3, 128, False, "nearest-even"), (6, 128, True, "nearest-even")])
def test_compile_time_schemes_vs_oracle(bits, g, sym, rnd, mode):
    """Symmetric / ceil / odd-bit schemes on the compile-time (streaming) kernels,
    bit-exact against the oracle: outputs and both stages' wire messages."""
    n, m = 4, 4 * 8192 * 5 + 4 * 24
    rng = np.random.default_rng(bits * 31 + g)
    xs = [(rng.standard_normal(m) * 3).astype(np.float32) for _ in range(n)]
    for x in xs:
        x[::301] *= 25
    xs = [orc.round_to_bf16(x) for x in xs]  # the GPU sees exactly these bf16 values
    codec = fc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)
    cfg = fc.FlashConfig.uniform(codec)
    comm = _comm(n, -(-m // n), cfg, mode)
    ts = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in xs]
    run = fc.flash_all_reduce(ts, cfg, comm=comm, out_dtype=torch.float32)
    oc = orc.Codec(bits=bits, group_size=g, symmetric=sym, rounding=rnd)
    res = orc.flash_all_reduce(xs, oc, oc)
    for o in run.outputs:
        assert np.array_equal(_bits(o.cpu().numpy()), _bits(res.outputs[0]))
    for j in range(n):
        p = (j + 1) % n
        assert comm.slot(p, 2, j, codec).to_bytes() == res.stage2[j].wire_bytes(), f"stage-2 {j}"
        s = (j + 1) % n
        if mode == "split":
            assert comm.slot(j, 1, s, codec).to_bytes() == res.stage1[j][s].wire_bytes(), f"stage-1 {j}<-{s}"
    comm.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("codec", [dict(bits=4), dict(bits=4, symmetric=True), dict(bits=4, rounding="ceil"),
                                   dict(bits=8), dict(bits=8, symmetric=True)])
def test_group_lane_kernels_match_lane_kernels(tp, codec):
    """g128 whole tiles take the 2-lanes-per-group reduce (and, for INT4, the
    group-per-lane scatter) — compiled for 16-bit outputs only, so the outputs
    here are bf16/fp16 (compared as int16). FC_OPT_STREAM_MASK bits 6/7 force
    the 32-element lane kernels: bit-identical. ~1800 tiles per call give every
    CTA of the persistent grids several tiles (ring slot / phase wrap-around at
    k >= 1, 2, 3), and the first 16 tiles of segment 0 (CTA 0's k = 0..3) are
    checked bit-exactly against the oracle."""
    tiles = -(-1800 // tp)
    m = tp * 8192 * tiles
    cfg = fc.FlashConfig.uniform(fc.CodecConfig(**codec))
    comm = _comm(tp, m // tp, cfg, "split")
    oc = orc.Codec(bits=codec["bits"], symmetric=codec.get("symmetric", False),
                   rounding=codec.get("rounding", "nearest-even"))
    for dt in (torch.bfloat16, torch.float16):
        g = torch.Generator(device="cuda").manual_seed(tp)
        ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(dt) for r in range(tp)]
        ts[0][5000:5128] = 1000.0  # a constant group (scale floor) and a large-offset one
        ts[1][9000:9128] += 3000.0
        outs = {}
        for mask in (0, 64 | 128):
            comm.set_option(_lib.OPT_STREAM_MASK, mask)
            outs[mask] = [o.clone() for o in comm.all_reduce_local(ts, cfg)]
        comm.set_option(_lib.OPT_STREAM_MASK, 0)
        for a, b in zip(outs[0], outs[64 | 128]):
            assert a.dtype == dt and torch.equal(a.view(torch.int16), b.view(torch.int16))
        seg, L = m // tp, 16 * 8192
        xr = [t[:L].float().cpu().numpy() for t in ts]  # segment 0's first 16 tiles of every rank
        red = orc.sequential_sum([orc.dequantize(orc.quantize(x, oc)) for x in xr])
        ref = torch.from_numpy(orc.dequantize(orc.quantize(red, oc))).to(dt)
        for r in (0, tp - 1):
            assert torch.equal(outs[0][r][:L].cpu().view(torch.int16), ref.view(torch.int16)), (dt, r)
    comm.close()


@pytest.mark.parametrize("tp", [2, 4, 8])
@pytest.mark.parametrize("codec", [dict(bits=4), dict(bits=4, symmetric=True), dict(bits=4, rounding="ceil"),
                                   dict(bits=8), dict(bits=8, symmetric=True)])
def test_fused_kernel_vs_split_and_oracle(tp, codec):
    """The fused single-launch kernel (k_fstream: group-lane scatter / reduce /
    gather roles, per-tile flags) for every schedule chunking — the whole
    segment, 1 tile, 3 tiles, an uneven split — is bit-identical to the
    phase-split kernels, and its stage-1 / stage-2 slots and outputs equal the
    oracle (bf16 and fp16, 16-bit outputs)."""
    tiles = 40
    m = tp * 8192 * tiles
    cfg = fc.FlashConfig.uniform(fc.CodecConfig(**codec))
    comm = _comm(tp, m // tp, cfg, "split")
    oc = orc.Codec(bits=codec["bits"], symmetric=codec.get("symmetric", False),
                   rounding=codec.get("rounding", "nearest-even"))
    try:
        for dt in (torch.bfloat16, torch.float16):
            g = torch.Generator(device="cuda").manual_seed(17 * tp + codec["bits"])
            ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(dt) for r in range(tp)]
            ts[0][5000:5128] = 1000.0
            comm.set_option(_lib.OPT_FUSED, 0)
            ref = [o.clone() for o in comm.all_reduce_local(ts, cfg)]
            comm.set_option(_lib.OPT_FUSED, 1)
            for chunk in (0, 1, 3, 17):
                comm.set_option(_lib.OPT_FUSED_CHUNK, chunk)
                for _ in range(2):  # back-to-back calls (epoch flags, no reset)
                    outs = comm.all_reduce_local(ts, cfg)
                    for r in range(tp):
                        assert torch.equal(outs[r].view(torch.int16), ref[r].view(torch.int16)), (dt, chunk, r)
            comm.set_option(_lib.OPT_FUSED_CHUNK, 0)
            xr = [t.float().cpu().numpy() for t in ts]
            res = orc.flash_all_reduce(xr, oc, oc)
            want = torch.from_numpy(res.outputs[0]).to(dt).view(torch.int16)
            assert torch.equal(outs[tp - 1].cpu().view(torch.int16), want)
            if dt == torch.bfloat16:
                for j in range(tp):
                    s = (j + 1) % tp
                    assert comm.slot(j, 1, s, cfg.stage1_codec).to_bytes() == res.stage1[j][s].wire_bytes()
                    assert comm.slot(s, 2, j, cfg.stage2_codec).to_bytes() == res.stage2[j].wire_bytes()
    finally:
        comm.close()


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("bs", [1, 8, 64])
def test_small_message_kernel_vs_oracle(bits, bs):
    """The one-launch small-message kernel (k_small; the default across GPUs for
    decode-sized rounds), forced on one GPU with OPT_ONESHOT 2: TP=8, bs x 8192
    bf16 per rank, bit-exact against the oracle, three calls in a row (the
    in-kernel epoch bump)."""
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    tp, m = 8, bs * 8192
    xs = orc.gen_rank_activations(8192, bs, bits, tp)
    xs = [orc.round_to_bf16(x.ravel()) for x in xs]
    cfg = fc.FlashConfig.from_bits(bits)
    oc = orc.Codec(bits=bits)
    want = orc.flash_all_reduce(xs, oc, oc).outputs[0]
    comm = FlashComm.local([0] * tp, slot_bytes_for(-(-m // tp), cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_ONESHOT, 2)
    ts = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in xs]
    for _ in range(3):
        outs = comm.all_reduce_local(ts, cfg, out_dtype=torch.float32)
        for o in outs:
            assert np.array_equal(o.cpu().numpy().view(np.uint32), want.view(np.uint32))
    assert comm.get_option(_lib.OPT_LAST_LAUNCHES) == 1
    comm.close()


@pytest.mark.parametrize("codec", [dict(bits=4), dict(bits=8), dict(bits=4, symmetric=True),
                                   dict(bits=8, symmetric=True), dict(bits=4, rounding="ceil")])
def test_fused_kernel_matches_split_multi_tile(codec):
    """The fused kernel (k_fstream: dynamic item dealing, per-tile flags, batched
    flag publishing, chunked schedules) is bit-identical to the phase-split
    kernels at TP=8 over 48 tiles per segment, for schedule chunks 1 / 2 / auto,
    repeated calls (tools/fused_stress.py runs the same over more calls)."""
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    tp, m = 8, 8 * 8192 * 48
    cfg = fc.FlashConfig.uniform(fc.CodecConfig(**codec))
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    g = torch.Generator(device="cuda").manual_seed(codec["bits"])
    ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(torch.bfloat16) for r in range(tp)]
    comm.set_option(_lib.OPT_FUSED, 0)
    ref = [o.clone() for o in comm.all_reduce_local(ts, cfg)]
    comm.set_option(_lib.OPT_FUSED, 1)
    for chunk in (1, 2, 0):
        comm.set_option(_lib.OPT_FUSED_CHUNK, chunk)
        for _ in range(3):
            outs = comm.all_reduce_local(ts, cfg)
            for a, b in zip(outs, ref):
                assert torch.equal(a.view(torch.int16), b.view(torch.int16)), chunk
    comm.close()


@pytest.mark.parametrize("codec", [dict(bits=4), dict(bits=8), dict(bits=4, symmetric=True),
                                   dict(bits=8, symmetric=True)])
def test_reduce_kernel_deterministic(codec):
    """The reduce kernel alone (FC_OPT_PHASES 2) on fixed receive slots gives the
    same stage-2 bytes every time (the piece-ring release race of DESIGN.md
    section 9 item 26 made INT8 sym non-deterministic at four CTAs per SM)."""
    from paper_2412_04964_b200 import _lib
    from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for

    tp = 8
    m = tp * 8192 * 225
    cc = fc.CodecConfig(**codec)
    cfg = fc.FlashConfig.uniform(cc)
    comm = FlashComm.local([0] * tp, slot_bytes_for(m // tp, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, 0)
    g = torch.Generator(device="cuda").manual_seed(tp)
    ts = [(torch.randn(m, device="cuda", generator=g) * (1 + r)).to(torch.bfloat16) for r in range(tp)]
    ts[0][5000:5128] = 1000.0
    ts[1][9000:9128] += 3000.0
    comm.all_reduce_local(ts, cfg)
    comm.set_option(_lib.OPT_PHASES, 2)
    runs = []
    for _ in range(4):
        comm.all_reduce_local(ts, cfg)
        runs.append([comm.slot((j + 1) % tp, 2, j, cc).to_bytes() for j in range(tp)])
    comm.set_option(_lib.OPT_PHASES, 0)
    comm.close()
    assert all(r == runs[0] for r in runs[1:])
