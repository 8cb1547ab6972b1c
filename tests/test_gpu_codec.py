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
    assert np.array_equal(q.scales[lo // 128: hi // 128].cpu().numpy().view(np.uint16), oq.scales.view(np.uint16))
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
    with pytest.raises(fc.IntegrityError):
        fc.dequantize(fc.QuantizedTensor.from_bytes(bytes(blob), 8, cfg), validate=True)


def test_known_answers():
    # test_codec.py:72-90
    q = fc.quantize(torch.arange(16, dtype=torch.float32, device="cuda"), fc.CodecConfig(bits=4, group_size=16))
    assert orc.unpack(q.codes.cpu().numpy(), 16, 4).tolist() == list(range(16))
    assert torch.equal(fc.dequantize(q).cpu(), torch.arange(16, dtype=torch.float32))
    q = fc.quantize(torch.tensor([-2.0, 2.0], device="cuda"), fc.CodecConfig(bits=4, group_size=2))
    assert orc.unpack(q.codes.cpu().numpy(), 2, 4).tolist() == [0, 15]
    assert int(q.zeros[0]) == 8
