"""GPU parity of the lane-8 path (csrc/fc_l8.cuh): group-scaled minifloat
codecs through the native cvt.rn.satfinite conversions (codec.py:332-351,
minifloat.py:58-118) and the Hadamard rotation fused into the flash
all-reduce's prologue / epilogue (rotation.py:38-83, collectives.py:350-351,
390-391), bit-exact against the oracle restatement (pinned to the reference's
own outputs by tests/test_oracle_golden.py and tests/golden/extras.npz)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import flash_oracle as orc

pytestmark = pytest.mark.gpu

fc = pytest.importorskip("paper_2412_04964_b200")
from paper_2412_04964_b200 import _lib  # noqa: E402
from paper_2412_04964_b200.comm import FlashComm, slot_bytes_for  # noqa: E402

FMTS = ("e4m3", "e5m2", "e2m1")


def _grid_sweep(fmt: str) -> np.ndarray:
    """Every grid magnitude, the midpoints between neighbours (ties), their f32
    neighbours on both sides, values past the largest finite one (saturation),
    the subnormal range down to below half the smallest subnormal, both signs
    (negative values that round to zero: encode() stores them as +0). Each
    128-group starts with +max_finite, so its scale is exactly 1."""
    f = orc.MINIFLOATS[fmt]
    tab = orc.mf_table(f).astype(np.float64)
    grid = np.unique(np.abs(tab[np.isfinite(tab)]))
    mids = (grid[:-1] + grid[1:]) / 2
    vals = [grid, mids, np.nextafter(mids.astype(np.float32), np.float32(0)),
            np.nextafter(mids.astype(np.float32), np.float32(np.inf)),
            np.array([f.max_finite * 1.02, f.max_finite * 1.5, f.max_finite * 4, f.sub_quantum / 2,
                      f.sub_quantum / 2 * 0.999, f.sub_quantum / 4, 1e-30, 0.0])]
    v = np.concatenate(vals).astype(np.float32)
    v = np.concatenate([v, -v])
    per = 127
    groups = -(-v.size // per)
    v = np.concatenate([v, np.zeros(groups * per - v.size, np.float32)]).reshape(groups, per)
    head = np.full((groups, 1), np.float32(f.max_finite))
    return np.concatenate([head, v], axis=1).ravel()


@pytest.mark.parametrize("fmt", FMTS)
def test_minifloat_grid_sweep_vs_oracle(fmt):
    x = _grid_sweep(fmt)
    cfg = fc.CodecConfig(number_format=fmt, group_size=128)
    q = fc.quantize(torch.from_numpy(x).cuda(), cfg)
    oq = orc.quantize(x, orc.Codec(kind=fmt, group_size=128))
    assert q.to_bytes() == oq.wire_bytes()
    d = fc.dequantize(q).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), orc.dequantize(oq).view(np.uint32))


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("g", [32, 64, 256])
def test_minifloat_random_groups_vs_oracle(fmt, g):
    rng = np.random.default_rng(g)
    x = (rng.standard_normal(8 * g * 37 + 5) * np.exp(rng.uniform(-8, 8, 8 * g * 37 + 5))).astype(np.float32)
    for dt in (torch.float32, torch.bfloat16, torch.float16):
        t = torch.from_numpy(x).to(dt).cuda()
        xr = t.float().cpu().numpy()
        q = fc.quantize(t, fc.CodecConfig(number_format=fmt, group_size=g))
        oq = orc.quantize(xr, orc.Codec(kind=fmt, group_size=g))
        assert q.to_bytes() == oq.wire_bytes(), dt


def _flash_case(n, m, st1, st2, rot, out_dtype, seed=0, ragged=0):
    xs = orc.gen_rank_activations(8192, -(-(m + ragged) // 8192), seed, n)
    xs = [orc.round_to_bf16(x.ravel()[: m + ragged]) for x in xs]
    oc = lambda s: orc.Codec(kind=s[0], group_size=s[1]) if isinstance(s[0], str) else orc.Codec(  # noqa: E731
        bits=s[0], group_size=s[1], symmetric=s[2])
    fcc = lambda s: fc.CodecConfig(number_format=s[0], group_size=s[1]) if isinstance(s[0], str) else \
        fc.CodecConfig(bits=s[0], group_size=s[1], symmetric=s[2])  # noqa: E731
    orot = None if rot is None else orc.Hadamard(*rot)
    res = orc.flash_all_reduce(xs, oc(st1), oc(st2), rotation=orot)
    cfg = fc.FlashConfig(fcc(st1), fcc(st2), rotation=None if rot is None else fc.HadamardBlock(*rot))
    seg = -(-(m + ragged) // n)
    comm = FlashComm.local([0] * n, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    ts = [torch.from_numpy(x).cuda().to(torch.bfloat16) for x in xs]
    run = fc.flash_all_reduce(ts, cfg, comm=comm, out_dtype=out_dtype)
    want = res.outputs[0]
    for o in run.outputs:
        if out_dtype == torch.float32:
            assert np.array_equal(o.cpu().numpy().view(np.uint32), want.view(np.uint32))
        else:
            assert np.array_equal(o.view(torch.int16).cpu().numpy(), orc.f32_to_bf16_bits(want).view(np.int16))
    if rot is None:  # stage buffers: bit-exact wire messages of both stages
        assert comm.slot(1, 1, 0, cfg.stage1_codec).to_bytes() == res.stage1[1][0].wire_bytes()
        assert comm.slot(0, 2, 3 % n, cfg.stage2_codec).to_bytes() == res.stage2[3 % n].wire_bytes()
    comm.close()


@pytest.mark.parametrize("st1,st2", [(("e4m3", 128), ("e4m3", 128)), (("e2m1", 32), ("e4m3", 32)),
                                     (("e5m2", 64), ("e5m2", 64)), (("e2m1", 128), ("e2m1", 128))])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_flash_minifloat_l8_vs_oracle(st1, st2, out_dtype):
    _flash_case(8, 8 * 8192 * 3, st1, st2, None, out_dtype)


@pytest.mark.parametrize("st,rot", [((4, 128, False), (128, True, None)), ((4, 128, False), (128, True, 7)),
                                    (("e4m3", 128), (64, False, 3)), ((8, 64, True), (256, True, 11)),
                                    ((4, 32, False), (8, True, 1))])
@pytest.mark.parametrize("ragged", [0, 128])
def test_flash_fused_rotation_vs_oracle(st, rot, ragged):
    """The rotation fused into the lane-8 kernels (no float32 copies of the
    rank tensors), at TP=4; a ragged M (segment 16416 elements: the zero
    padding is rotated with the data) fuses for an 8-element block and takes
    the three-pass fallback for larger ones."""
    n, m = 4, 4 * 8192 * 2
    seg = -(-(m + ragged) // n)
    if (n * seg) % rot[0]:
        pytest.skip("the reference itself rejects this length (rotation.py:52-58)")
    comm_probe = FlashComm.local([0] * n, 1 << 20)
    fcc = fc.CodecConfig(number_format=st[0], group_size=st[1]) if isinstance(st[0], str) else \
        fc.CodecConfig(bits=st[0], group_size=st[1], symmetric=st[2])
    assert comm_probe.rotation_fusable(m + ragged, fc.FlashConfig.uniform(fcc), fc.HadamardBlock(*rot)) == \
        (seg % rot[0] == 0 and seg % st[1] == 0)
    comm_probe.close()
    _flash_case(n, m, st, st, rot, torch.float32, seed=2, ragged=ragged)


def test_minifloat_flash_ipc_free_path_launch_count():
    """A minifloat flash call is three lane-8 launches per round on one GPU."""
    n, m = 4, 4 * 8192
    cfg = fc.FlashConfig.uniform(fc.CodecConfig(number_format="e4m3"))
    comm = FlashComm.local([0] * n, slot_bytes_for(m // n, cfg.stage1_codec, cfg.stage2_codec))
    ts = [torch.randn(m, device="cuda").to(torch.bfloat16) for _ in range(n)]
    comm.all_reduce_local(ts, cfg)
    assert comm.get_option(_lib.OPT_LAST_LAUNCHES) == 3
    comm.close()


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("g", [64, 128, 256])
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
def test_minifloat_streaming_codec_vs_oracle(fmt, g, dt):
    """16-bit inputs, whole tiles: the minifloat codec on the TMA-fed streaming
    kernels (k_qstream_gpl<MfSpec> / k_dstream<MfSpec>), bit-exact against the
    oracle: random groups over 16 binades plus the grid sweep (ties, subnormals,
    saturation) rounded to the input dtype."""
    rng = np.random.default_rng(g)
    n = 8192 * 5
    x = (rng.standard_normal(n) * np.exp(rng.uniform(-6, 6, n))).astype(np.float32)
    sw = _grid_sweep(fmt)
    if dt == torch.float16:  # e5m2 saturation probes exceed the fp16 range (inf would be a DomainError)
        sw = np.clip(sw, -60000.0, 60000.0)
    x[: sw.size] = sw
    t = torch.from_numpy(x).to(dt).cuda()
    xr = t.float().cpu().numpy()
    cc = fc.CodecConfig(number_format=fmt, group_size=g)
    q = fc.quantize(t, cc)
    oq = orc.quantize(xr, orc.Codec(kind=fmt, group_size=g))
    assert q.to_bytes() == oq.wire_bytes()
    for odt in (torch.float32, dt):
        d = fc.dequantize(q, dtype=odt).float().cpu().numpy()
        want = torch.from_numpy(orc.dequantize(oq)).to(odt).float().numpy()
        assert np.array_equal(d.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("fmt", FMTS)
@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("slot_tiles", [0, 1])
def test_flash_minifloat_streaming_vs_oracle(fmt, dt, slot_tiles):
    """One minifloat format in both stages, g = 128, 16-bit in and out: the TMA-fed streaming
    kernels (k_qstream_gpl / k_rstream_gpl / k_dstream on MfSpec) -- one round, or three
    rounds of one tile (slots sized for one tile) -- bit-exact against the oracle, stage
    buffers included, and equal to the fused kernel and the lane-8 kernels (FC_OPT_STREAM_MASK
    bit 10)."""
    n, tiles = 8, 3
    m = n * 8192 * tiles
    rng = np.random.default_rng(7)
    xs = [(rng.standard_normal(m) * np.exp(rng.uniform(-3, 3, m))).astype(np.float32) for _ in range(n)]
    ts = [torch.from_numpy(x).to(dt) for x in xs]
    xs = [t.float().numpy() for t in ts]
    oc = orc.Codec(kind=fmt, group_size=128)
    res = orc.flash_all_reduce(xs, oc, oc)
    cc = fc.CodecConfig(number_format=fmt, group_size=128)
    cfg = fc.FlashConfig.uniform(cc)
    seg = m // n
    comm = FlashComm.local([0] * n, slot_bytes_for(8192 if slot_tiles else seg, cc, cc))
    dts = [t.cuda() for t in ts]
    want = torch.from_numpy(res.outputs[0]).to(dt).view(torch.int16).numpy()
    run = fc.flash_all_reduce(dts, cfg, comm=comm, out_dtype=dt)
    launches = comm.get_option(_lib.OPT_LAST_LAUNCHES)  # three per round
    assert launches == 3 if not slot_tiles else (launches % 3 == 0 and launches >= 6)
    for o in run.outputs:
        assert np.array_equal(o.view(torch.int16).cpu().numpy(), want)
    if not slot_tiles:
        assert comm.slot(1, 1, 0, cc).to_bytes() == res.stage1[1][0].wire_bytes()
        assert comm.slot(0, 2, 3, cc).to_bytes() == res.stage2[3].wire_bytes()
    comm.set_option(_lib.OPT_FUSED, 1)  # the single-launch fused kernel on MfSpec (cross-GPU default)
    runf = fc.flash_all_reduce(dts, cfg, comm=comm, out_dtype=dt)
    fl = comm.get_option(_lib.OPT_LAST_LAUNCHES)
    assert fl == 2 * launches // 3, (fl, launches)  # epoch bump + k_fstream per round
    comm.set_option(_lib.OPT_FUSED, -1)
    comm.set_option(_lib.OPT_STREAM_MASK, 1024)
    run2 = fc.flash_all_reduce(dts, cfg, comm=comm, out_dtype=dt)
    for o, o2, o3 in zip(run.outputs, run2.outputs, runf.outputs):
        assert torch.equal(o.view(torch.int16), o2.view(torch.int16))
        assert torch.equal(o.view(torch.int16), o3.view(torch.int16))
    comm.close()
