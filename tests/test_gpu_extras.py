"""GPU parity of SURVEY §8f row 4: group-scaled minifloat stage codecs
(e4m3 / e5m2 / e2m1, codec.py:332-351) and the Hadamard rotation
(rotation.py:61-83, collectives.py:350-351,390-391), bit-exact against the
reference's own outputs (tests/golden/extras.npz)."""

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


def _stage(spec):
    if isinstance(spec, (list, tuple)) and isinstance(spec[0], str):
        return fc.CodecConfig(number_format=spec[0], group_size=spec[1])
    if spec == "fp16":
        return fc.PASSTHROUGH_FP16
    bits, g, sym, rnd = spec
    return fc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)


@pytest.mark.parametrize("i", range(len(gio.extras_meta()["minifloat"])))
def test_minifloat_codec_golden(i):
    z, m = gio.extras_npz(), gio.extras_meta()["minifloat"][i]
    cfg = fc.CodecConfig(number_format=m["format"], group_size=m["group_size"])
    x = torch.from_numpy(z[f"mf{i}_x"]).cuda()
    q = fc.quantize(x, cfg)
    assert q.to_bytes() == bytes(z[f"mf{i}_wire"])
    d = fc.dequantize(q).cpu().numpy()
    assert np.array_equal(d.view(np.uint32), z[f"mf{i}_deq"].view(np.uint32))


@pytest.mark.parametrize("mode", ["split", "fused"])
@pytest.mark.parametrize("i", range(len(gio.extras_meta()["flash"])))
def test_flash_minifloat_rotation_golden(i, mode):
    z, m = gio.extras_npz(), gio.extras_meta()["flash"][i]
    n = m["n"]
    xs = [z[f"fl{i}_x{r}"] for r in range(n)]
    rot = None if m["rotation"] is None else fc.HadamardBlock(*m["rotation"])
    cfg = fc.FlashConfig(_stage(m["stage1"]), _stage(m["stage2"]), rotation=rot)
    seg = -(-m["m"] // n)
    comm = FlashComm.local([0] * n, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_option(_lib.OPT_FUSED, 1 if mode == "fused" else 0)
    ts = [torch.from_numpy(x).cuda() for x in xs]
    run = fc.flash_all_reduce(ts, cfg, comm=comm, out_dtype=torch.float32)
    want = z[f"fl{i}_out"]
    for o in run.outputs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want.view(np.uint32)), m
    assert run.wire_bytes_per_rank == m["wire_bytes_per_rank"]
    comm.close()


def test_hadamard_roundtrip_and_errors():
    rng = np.random.default_rng(5)
    x = rng.standard_normal(4096).astype(np.float32)
    for blk in (fc.HadamardBlock(64), fc.HadamardBlock(128, sign_seed=9), fc.HadamardBlock(32, normalize=False)):
        t = torch.from_numpy(x).cuda()
        y = fc.hadamard_apply(t, blk)
        oh = orc.Hadamard(blk.dimension, blk.normalize, blk.sign_seed)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), orc.hadamard_apply(x, oh).view(np.uint32))
        back = fc.hadamard_inverse(y, blk).cpu().numpy()
        assert np.array_equal(back.view(np.uint32), orc.hadamard_inverse(orc.hadamard_apply(x, oh), oh).view(np.uint32))
    with pytest.raises(fc.DomainError):
        fc.hadamard_apply(torch.zeros(100, device="cuda"), fc.HadamardBlock(64))
    with pytest.raises(fc.ConfigError):
        fc.HadamardBlock(48)
