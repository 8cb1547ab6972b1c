"""GPU parity of the single-GPU codec kernels (fc_quantize / fc_dequantize)
against the reference's golden vectors and the oracle. Bit-exact: codes,
fp16 scales, zeros, wire bytes and float32 dequantized values."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import flash_oracle as orc
from tests import golden_io as gio

pytestmark = pytest.mark.gpu

fc = pytest.importorskip("paper_2412_04964_b200")


def _cfg(meta) -> "fc.CodecConfig":
    if meta.get("kind") == "fp16":
        return fc.PASSTHROUGH_FP16
    return fc.CodecConfig(bits=meta["bits"], group_size=meta["group_size"], symmetric=meta["symmetric"],
                          rounding=meta["rounding"])


@pytest.mark.parametrize("i", range(len(gio.codec_meta())))
def test_codec_golden(i):
    z = gio.codec_npz()
    meta = gio.codec_meta()[i]
    cfg = _cfg(meta)
    x = torch.from_numpy(z[f"x{i}"]).cuda()
    q = fc.quantize(x, cfg)
    assert q.to_bytes() == bytes(z[f"wire{i}"])
    d = fc.dequantize(q).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), z[f"deq{i}"].view(np.uint32))


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("bits,g,sym,rnd", [(4, 128, False, "nearest-even"), (8, 128, False, "nearest-even"),
                                            (4, 32, True, "ceil"), (8, 256, True, "nearest-even"),
                                            (2, 64, False, "ceil"), (6, 64, False, "nearest-even")])
def test_codec_half_inputs_vs_oracle(dtype, bits, g, sym, rnd):
    rng = np.random.default_rng(bits * 1000 + g)
    n = 3 * 8192 + 777
    x32 = (rng.standard_normal(n) * 4).astype(np.float32)
    x32[::97] *= 40
    t = torch.from_numpy(x32).cuda().to(dtype)
    xr = t.float().cpu().numpy()
    cfg = fc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)
    q = fc.quantize(t, cfg)
    oq = orc.quantize(xr, orc.Codec(bits=bits, group_size=g, symmetric=sym, rounding=rnd))
    assert q.to_bytes() == oq.wire_bytes()
    for odt in (torch.float32, torch.bfloat16, torch.float16):
        d = fc.dequantize(q, dtype=odt).float().cpu().numpy()
        ref = orc.dequantize(oq)
        ref = torch.from_numpy(ref).to(odt).float().numpy()
        assert np.array_equal(d.view(np.uint32), ref.view(np.uint32))


def test_large_c5_shape_bitexact_sample():
    # C5: bf16 [8,1024,8192] int4 g128; check a 1M-element window exactly
    torch.manual_seed(0)
    x = torch.randn(8, 1024, 8192, device="cuda", dtype=torch.bfloat16)
    cfg = fc.CodecConfig(bits=4)
    q = fc.quantize(x, cfg)
    lo, hi = 5 * 2 ** 20, 6 * 2 ** 20
    xs = x.reshape(-1)[lo:hi].float().cpu().numpy()
    oq = orc.quantize(xs, orc.Codec(bits=4))
    assert np.array_equal(q.codes[lo // 2: hi // 2].cpu().numpy(), orc.pack(oq.codes, 4))
    assert np.array_equal(q.scales_f16[lo // 128: hi // 128].cpu().numpy().view(np.uint16), oq.scales.view(np.uint16))
    assert np.array_equal(q.zeros[lo // 128: hi // 128].cpu().numpy(), oq.zeros)


def test_nonfinite_raises_domain_error():
    x = torch.randn(5000, device="cuda")
    x[1234] = float("nan")
    with pytest.raises(fc.DomainError):
        fc.quantize(x, fc.CodecConfig(bits=4))
    x[1234] = float("inf")
    with pytest.raises(fc.DomainError):
        fc.quantize(x, fc.CodecConfig(bits=8, group_size=96))


def test_empty_raises_domain_error():
    with pytest.raises(fc.DomainError):
        fc.quantize(torch.empty(0, device="cuda"), fc.CodecConfig(bits=4))


def test_wire_roundtrip_and_integrity():
    x = torch.randn(500, device="cuda") * 3
    for name in ("int4asym", "int4sym", "int8asym", "int8sym", "fp16"):
        cfg = fc.codec_from_name(name, group_size=32)
        q = fc.quantize(x, cfg)
        blob = q.to_bytes()
        assert len(blob) == cfg.wire_byte_len(500) == q.wire_bytes
        q2 = fc.QuantizedTensor.from_bytes(blob, 500, cfg)
        assert torch.equal(fc.dequantize(q), fc.dequantize(q2))
    with pytest.raises(fc.IntegrityError):
        fc.QuantizedTensor.from_bytes(b"\x00" * 7, 16, fc.CodecConfig(bits=4, group_size=16))
    # codec.py:373-374 tampered 2-bit codes
    cfg = fc.CodecConfig(bits=2, group_size=8)
    blob = bytearray(fc.quantize(torch.linspace(-1, 1, 8, device="cuda"), cfg).to_bytes())
    blob[0] = 0xFF
    with pytest.raises(fc.IntegrityError):  # validated by default, like codec.py:354-384
        fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 8, cfg))
    fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 8, cfg), validate=False)  # opt-out: no check
    # test_codec.py:157-163: non-positive / non-finite scales
    cfg = fc.CodecConfig(bits=4, group_size=8)
    q = fc.quantize(torch.linspace(-1, 1, 16, device="cuda"), cfg)
    for bad in (0.0, -1.0, float("inf"), float("nan")):
        blob = bytearray(q.to_bytes())
        blob[8:10] = np.array([bad], np.float16).tobytes()
        with pytest.raises(fc.IntegrityError):
            fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 16, cfg))
    # zero point past the 2^bits - 1 range (3-bit codec, zero byte 9)
    cfg = fc.CodecConfig(bits=3, group_size=8)
    blob = bytearray(fc.quantize(torch.linspace(-1, 1, 8, device="cuda"), cfg).to_bytes())
    blob[-1] = 9
    with pytest.raises(fc.IntegrityError):
        fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 8, cfg))
    # the padding nibble of an odd count is not a code (bitpack.py:64-75)
    cfg = fc.CodecConfig(bits=2, group_size=8)
    blob = bytearray(fc.quantize(torch.linspace(-1, 1, 7, device="cuda"), cfg).to_bytes())
    blob[3] |= 0xF0
    fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 7, cfg))


def test_known_answers():
    # test_codec.py:72-90
    q = fc.quantize(torch.arange(16, dtype=torch.float32, device="cuda"), fc.CodecConfig(bits=4, group_size=16))
    assert orc.unpack(q.codes.cpu().numpy(), 16, 4).tolist() == list(range(16))
    assert torch.equal(fc.dequantize(q).cpu(), torch.arange(16, dtype=torch.float32))
    q = fc.quantize(torch.tensor([-2.0, 2.0], device="cuda"), fc.CodecConfig(bits=4, group_size=2))
    assert orc.unpack(q.codes.cpu().numpy(), 2, 4).tolist() == [0, 15]
    assert int(q.zeros[0]) == 8


def _adversarial(n, dtype, seed):
    """Groups that take every branch of the lane codecs: a large offset with a
    tiny spread (|x/s| >= 2^14: the float-clamp path), constant groups (scale
    floor), fp16-overflowing ranges (scale 65504), tiny values (floor bump),
    signed zeros, next to ordinary groups inside the same warp."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n).astype(np.float32)
    g = 128
    for k in range(n // g):
        kind = k % 8
        sl = slice(k * g, (k + 1) * g)
        if kind == 1:
            x[sl] = 1000.0 + rng.standard_normal(g).astype(np.float32) * 0.01
        elif kind == 2:
            x[sl] = -3.5
        elif kind == 3:
            x[sl] = rng.uniform(-60000, 60000, g).astype(np.float32) * (1e5 if dtype == torch.bfloat16 else 1.0)
        elif kind == 4:
            x[sl] = rng.standard_normal(g).astype(np.float32) * 1e-9
        elif kind == 5:
            x[sl] = np.where(rng.random(g) < 0.5, -0.0, 0.0).astype(np.float32)
        elif kind == 6:
            x[sl] = -77.0 - np.abs(rng.standard_normal(g).astype(np.float32)) * 1e-3
    return torch.from_numpy(x).to(dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("bits,g,sym,rnd", [(4, 128, False, "nearest-even"), (8, 128, False, "nearest-even"),
                                            (4, 128, True, "nearest-even"), (4, 128, False, "ceil"),
                                            (8, 128, True, "ceil"), (4, 64, False, "nearest-even")])
def test_codec_adversarial_groups_vs_oracle(dtype, bits, g, sym, rnd):
    n = 4 * 8192 + 3 * 128 + 40  # whole tiles plus a ragged tail tile
    t = _adversarial(n, dtype, seed=bits + g)
    xr = t.float().numpy()
    cfg = fc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)
    q = fc.quantize(t.cuda(), cfg)
    oq = orc.quantize(xr, orc.Codec(bits=bits, group_size=g, symmetric=sym, rounding=rnd))
    assert q.to_bytes() == oq.wire_bytes()
    d = fc.dequantize(q, dtype=torch.float32).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), orc.dequantize(oq).view(np.uint32))


@pytest.mark.parametrize("bits", [4, 8])
def test_flash_adversarial_groups_vs_oracle(bits):
    n, m = 4, 4 * (2 * 8192 + 256)
    ts = [_adversarial(m, torch.bfloat16, seed=10 * r + bits) * (1 + r) for r in range(n)]
    ts = [t.to(torch.bfloat16) for t in ts]
    xr = [t.float().numpy() for t in ts]
    ref = orc.flash_all_reduce(xr, orc.Codec(bits=bits), orc.Codec(bits=bits)).outputs[0]
    run = fc.flash_all_reduce([t.cuda() for t in ts], fc.FlashConfig.from_bits(bits), out_dtype=torch.float32)
    for o in run.outputs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_quantized_tensor_reference_constructor():
    """QuantizedTensor(codes, scales, zeros, element_count, config) as in
    codec.py:165-181: float32 scales, shape checks -> IntegrityError, the wire
    bytes and the decode equal the oracle's."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal(1000).astype(np.float32)
    for oc, cc in ((orc.Codec(bits=4), fc.CodecConfig(bits=4)), (orc.Codec(bits=8, symmetric=True),
                   fc.CodecConfig(bits=8, symmetric=True)), (orc.Codec(kind="e4m3"), fc.CodecConfig(number_format="e4m3"))):
        oq = orc.quantize(x, oc)
        q = fc.QuantizedTensor(orc.pack(oq.codes, oc.storage_bits), oq.scales.astype(np.float32),
                               oq.zeros if cc.is_int and not cc.symmetric else None, x.size, cc)
        assert q.scales.dtype == torch.float32 and q.to_bytes() == oq.wire_bytes()
        assert np.array_equal(fc.dequantize(q).cpu().numpy().view(np.uint32), orc.dequantize(oq).view(np.uint32))
        with pytest.raises(fc.IntegrityError):
            fc.QuantizedTensor(np.zeros(1, np.uint8), oq.scales, None, x.size, cc)
        with pytest.raises(fc.IntegrityError):
            fc.QuantizedTensor(q.codes, oq.scales[:-1], q.zeros, x.size, cc)


def test_topology_nvml():
    from paper_2412_04964_b200.comm import FlashComm

    comm = FlashComm.local([0, 0], 1 << 16)
    t = comm.topology()
    comm.close()
    assert t["world_size"] == 2 and t["peer_access"][0][1] == 1 and "B200" in " ".join(t["device_names"])
    nv = t["nvlink"]
    assert nv["nvml"] and "0" in nv["devices"] and nv["devices"]["0"]["nvlink_active"] >= 0
