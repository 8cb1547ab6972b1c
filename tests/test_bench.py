"""bench.py host logic on CPU: the multi-GPU roofline against the reference's
own wire-byte formula (costmodel.py:122-128, SURVEY §8d floors), and the CPU
reference arm — the unmodified qcollectives.flash_all_reduce from
baseline/_ref and the oracle port — agreeing on the same inputs."""

from __future__ import annotations

import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_dist_roofline_c2_matches_survey_floor():
    # C2: TP=8, INT4 g128, bf16 8x1024x8192 per rank: 61.47 MB per direction -> 68.30 us at 900 GB/s
    m = 8 * 1024 * 8192
    seg = m // 8
    w = bench.wire_len(4, 128, seg)
    r = bench.dist_roofline(8, m, 2, w, w, 6453.4, 0.1)
    assert r["nvlink_bytes_per_rank"] == 61_472_768
    assert r["bound"] == "nvlink"
    assert abs(r["t_roof_us"] - 68.30) < 0.01
    assert r["peak"] == 900.0
    assert abs(r["frac"] - 0.6830) < 1e-3
    # TP=2 INT4 is HBM-bound (SURVEY: 51.7 us at 6550.7 GB/s)
    w2 = bench.wire_len(4, 128, m // 2)
    r2 = bench.dist_roofline(2, m, 2, w2, w2, 6550.7, 0.1)
    assert r2["bound"] == "hbm" and abs(r2["t_roof_us"] - 51.7) < 0.1


def test_wire_len_matches_reference_ledger():
    from oracle import flash_oracle as orc

    for bits in (4, 8):
        for n in (128, 8192, 1000):
            assert bench.wire_len(bits, 128, n) == orc.Codec(bits=bits).wire_len(n)


@pytest.mark.skipif(not bench.have_reference(), reason="baseline/_ref (the reference install) absent")
def test_cpu_reference_arm_agrees_with_port():
    cfg = dict(bench.CONFIGS["c2"])
    cfg["tp"] = 4
    ref = bench.CpuReference(cfg, 2, 1, kind="reference")
    port = bench.CpuReference(cfg, 2, 1, kind="port")
    try:
        for r in (ref, port):
            assert r.step(3) > 0
        a = ref.pool.map(bench._ref_call, [3000, 3001])
        b = port.pool.map(bench._ref_call, [3000, 3001])
        # same inputs (the reference's generator vs the oracle's restatement) -> same outputs
        assert [x[1] for x in a] == [x[1] for x in b]
        assert "unmodified qcollectives" in ref.describe()
    finally:
        ref.close()
        port.close()
