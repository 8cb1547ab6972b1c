"""CPU-side checks of the host layer and the C ABI (no GPU needed):
the library loads and exports every symbol include/flashcomm.h declares;
host-only entry points (validation, layouts, chunk resolution) match the
reference semantics; configs mirror the reference; the ledger equals the
reference's measured wire bytes."""

from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2412_04964_b200 as fc
from oracle import flash_oracle as orc
from paper_2412_04964_b200 import _lib
from tests import golden_io as gio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "flashcomm.h")) as fh:
        src = fh.read()
    return sorted(set(re.findall(r"FC_API\s+[\w\s\*]*?\b(fc_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 20
    L = _lib.lib()
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fc_\w+)", out))
    assert set(syms) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version():
    assert b"sm_100a" in _lib.lib().fc_version()


CODECS = [fc.CodecConfig(bits=b, group_size=g, symmetric=s)
          for b in (2, 3, 4, 5, 6, 7, 8) for g in (1, 3, 32, 96, 128, 256) for s in (False, True)]


@pytest.mark.parametrize("cfg", CODECS + [fc.PASSTHROUGH_FP16], ids=lambda c: f"{c.label}-g{c.group_size}")
def test_layout_matches_reference_wire_len(cfg):
    for n in (1, 2, 7, 128, 1000, 8192, 8192 * 3 + 5):
        L = cfg.device_layout(n)
        assert L.wire_bytes == cfg.wire_byte_len(n)
        oc = orc.FP16 if cfg.is_passthrough else orc.Codec(bits=cfg.bits, group_size=cfg.group_size,
                                                             symmetric=cfg.symmetric)
        assert L.wire_bytes == oc.wire_len(n)
        assert L.scales_offset % 16 == 0 and L.zeros_offset % 16 == 0
        assert L.scales_offset >= L.codes_bytes and L.total_bytes >= L.zeros_offset


def test_codec_validation_mirrors_reference():
    for kw in (dict(), dict(bits=4, number_format="e4m3"), dict(bits=1), dict(bits=9),
               dict(bits=4, group_size=0), dict(bits=4, rounding="up"), dict(bits=4, scale_floor=0.0),
               dict(number_format="e3m3")):
        with pytest.raises(fc.ConfigError):
            fc.CodecConfig(**kw)
    bad = _lib.fc_codec(_lib.KIND_INT, 9, 128, 0, 0, 0, 1e-8)
    assert _lib.lib().fc_codec_validate(C.byref(bad)) == 1
    mf = fc.CodecConfig(number_format="e4m3").to_fc()  # minifloats: kind 2, format id in `reserved`
    assert (mf.kind, mf.bits, mf.reserved) == (_lib.KIND_MINIFLOAT, 8, 0)
    assert _lib.lib().fc_codec_validate(C.byref(mf)) == 0
    bad_mf = _lib.fc_codec(_lib.KIND_MINIFLOAT, 8, 128, 0, 0, 7, 1e-8)
    assert _lib.lib().fc_codec_validate(C.byref(bad_mf)) == 1
    for fmt, wire in (("e4m3", 1000 + 8 * 2), ("e5m2", 1000 + 8 * 2), ("e2m1", 500 + 8 * 2)):
        cfg = fc.CodecConfig(number_format=fmt)
        assert cfg.device_layout(1000).wire_bytes == cfg.wire_byte_len(1000) == wire


def test_json_and_names():
    for cfg in (fc.CodecConfig(bits=4, group_size=64, symmetric=True, rounding="ceil"), fc.PASSTHROUGH_FP16):
        assert fc.CodecConfig.from_json_dict(cfg.to_json_dict()) == cfg
    with pytest.raises(fc.ConfigError):
        fc.CodecConfig.from_json_dict({"bits": 4, "tone": "mauve"})
    assert fc.codec_from_name("int4") == fc.CodecConfig(bits=4)
    assert fc.codec_from_name("fp16") is fc.PASSTHROUGH_FP16
    with pytest.raises(fc.ConfigError):
        fc.codec_from_name("int9000")
    s1, s2 = fc.int6_flash_pair(group_size=64)
    assert (s1.bits, s2.bits, s1.group_size) == (4, 8, 64)


@pytest.mark.parametrize("n", range(1, 9))
def test_resolve_chunk_matches_reference(n):
    for cfg in (fc.FlashConfig.from_bits(4), fc.FlashConfig.int6(group_size=96), fc.FlashConfig.from_bits(16),
                fc.FlashConfig(fc.CodecConfig(bits=4, group_size=32), fc.CodecConfig(bits=8, group_size=48))):
        c = _lib.fc_flash_cfg(cfg.stage1_codec.to_fc(), cfg.stage2_codec.to_fc(), 0)
        out = C.c_int64()
        assert _lib.lib().fc_flash_resolve_chunk(C.byref(c), n, C.byref(out)) == 0
        s1 = orc.FP16 if cfg.stage1_codec.is_passthrough else orc.Codec(bits=cfg.stage1_codec.bits,
                                                                          group_size=cfg.stage1_codec.group_size)
        s2 = orc.FP16 if cfg.stage2_codec.is_passthrough else orc.Codec(bits=cfg.stage2_codec.bits,
                                                                          group_size=cfg.stage2_codec.group_size)
        assert out.value == cfg.resolve_chunk_size(n) == orc.resolve_chunk(n, s1, s2)
    bad = fc.FlashConfig.from_bits(4, chunk_size=128)
    with pytest.raises(fc.ConfigError):
        bad.resolve_chunk_size(4)
    c = _lib.fc_flash_cfg(bad.stage1_codec.to_fc(), bad.stage2_codec.to_fc(), 128)
    assert _lib.lib().fc_flash_resolve_chunk(C.byref(c), 4, C.byref(C.c_int64())) == 1


@pytest.mark.parametrize("i", range(len(gio.flash_meta())))
def test_ledger_matches_reference_wire_bytes(i):
    meta = gio.flash_meta()[i]
    n, m = meta["n"], meta["m"]

    def st(spec):
        return fc.PASSTHROUGH_FP16 if spec == "fp16" else fc.CodecConfig(
            bits=spec[0], group_size=spec[1], symmetric=spec[2], rounding=spec[3])

    led = fc.flash_ledger(n, -(-m // n), meta["resolved_chunk"] // n, st(meta["stage1"]), st(meta["stage2"]))
    assert led.rank_bytes_sent(0) == meta["wire_bytes_per_rank"]
    # reference ledger: every directed pair carries the same bytes, 2 msgs per piece
    assert all(led.bytes_sent[s][r] == (0 if s == r else led.bytes_sent[0][1]) for s in range(n) for r in range(n))


def test_flash_config_presets():
    assert fc.FlashConfig.from_bits(16).stage1_codec.is_passthrough
    assert fc.FlashConfig.from_bits(6).stage2_codec.bits == 8
    with pytest.raises(fc.ConfigError):
        fc.FlashConfig.from_bits(5)
    with pytest.raises(fc.ConfigError):
        fc.FlashConfig.from_bits(4, chunk_size=0)
    with pytest.raises(fc.ConfigError):
        fc.run_collective("bogus", [np.zeros(4)])
    with pytest.raises(fc.ConfigError):
        fc.run_collective("ring", [np.zeros(4)])
    with pytest.raises(fc.ConfigError):
        fc.FabricTopology(world_size=0)


def test_comm_create_rejects_bad_world():
    h = C.c_void_p()
    devs = (C.c_int32 * 1)(0)
    assert _lib.lib().fc_comm_create_local(0, devs, 1 << 20, C.byref(h)) == 1
    assert _lib.lib().fc_comm_create_local(17, devs, 1 << 20, C.byref(h)) == 1
    assert _lib.lib().fc_comm_create_ipc(4, 5, 0, 1 << 20, C.byref(h)) == 1
