"""Generate golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package `qcollectives` from
/root/reference/pkg/src and records, on seeded inputs:

* codec.npz   — reference `quantize` codes/scales/zeros and `dequantize`
                outputs over bits 2..8, many group sizes, sym/asym,
                nearest/ceil and adversarial input families
                (codec.py:292-384).
* flash.npz   — reference `flash_all_reduce` outputs (rank 0; all ranks are
                checked identical here), `all_reduce_exact` outputs, and the
                reference's own wire messages captured from its fabric
                (`Fabric._send`, fabric.py:151-156), per (src, dst) in send
                order (collectives.py:321-402).
* reports.json — `rs_vs_ag_experiment` MSEs (workload.py:176-200) and the
                BASELINE.md §2 MSE table (flash vs exact, 1024x8192 bf16).

The fixtures are committed; nothing at GPU/test run time reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import qcollectives as qc  # noqa: E402  (reference, read-only)
from qcollectives import fabric as qfabric  # noqa: E402

from oracle.flash_oracle import round_to_bf16, round_to_fp16  # noqa: E402


# ---------------------------------------------------------------------------
# input families


def fam_inputs(rng: np.random.Generator, family: str, n: int) -> np.ndarray:
    if family == "gauss_bf16":
        return round_to_bf16((rng.standard_normal(n) * 3).astype(np.float32))
    if family == "outlier_fp16":
        x = rng.standard_normal(n).astype(np.float32)
        idx = rng.choice(n, size=max(1, n // 50), replace=False)
        x[idx] *= 30
        return round_to_fp16(x)
    if family == "stage2_sum":
        # realistic stage-2 input: sum of 8 dequantized int4 tensors
        cfg = qc.CodecConfig(bits=4, group_size=128)
        acc = np.zeros(n, np.float32)
        for _ in range(8):
            acc += qc.dequantize(qc.quantize(rng.standard_normal(n).astype(np.float32), cfg))
        return acc
    if family == "wide_exp":
        # exponents 2^-30..2^30, includes groups whose scale overflows fp16
        mag = np.exp2(rng.uniform(-30, 30, n)).astype(np.float32)
        return (mag * rng.choice([-1.0, 1.0], n)).astype(np.float32)
    if family == "degenerate":
        # constant groups, one-signed groups, zeros, tiny values (scale floor)
        x = rng.standard_normal(n).astype(np.float32)
        k = n // 5
        x[:k] = 5.0
        x[k:2 * k] = np.abs(x[k:2 * k]) + 1.0
        x[2 * k:3 * k] = 0.0
        x[3 * k:4 * k] = (rng.standard_normal(k) * 1e-9).astype(np.float32)
        return x
    if family == "near_ties":
        # values at and around (k + 1/2) * s for an fp16 scale s
        s = np.float32(np.float16(0.0371))
        k = rng.integers(-7, 8, n).astype(np.float32)
        x = ((k + 0.5) * s).astype(np.float32)
        jitter = rng.integers(-2, 3, n).astype(np.int32)
        x = (x.view(np.int32) + jitter).view(np.float32)
        x[0], x[1] = -8 * s, 7 * s  # pin group range to 15 * s
        return x
    raise ValueError(family)


FAMILIES = ["gauss_bf16", "outlier_fp16", "stage2_sum", "wide_exp", "degenerate", "near_ties"]


def codec_cases():
    cases = []
    for bits in range(2, 9):
        for g in (1, 3, 16, 32, 64, 96, 128, 256):
            for sym in (False, True):
                for rnd in ("nearest-even", "ceil"):
                    cases.append(dict(bits=bits, group_size=g, symmetric=sym, rounding=rnd))
    return cases


def make_codec(out_path: str) -> None:
    rng = np.random.default_rng(20241206)
    arrays = {}
    meta = []
    for i, c in enumerate(codec_cases()):
        fam = FAMILIES[i % len(FAMILIES)]
        n = int(rng.choice([997, 1024, 1500, 4096]))
        x = fam_inputs(rng, fam, n)
        cfg = qc.CodecConfig(bits=c["bits"], group_size=c["group_size"],
                             symmetric=c["symmetric"], rounding=c["rounding"])
        q = qc.quantize(x, cfg)
        arrays[f"x{i}"] = x
        arrays[f"codes{i}"] = qc.unpack(q.codes)
        arrays[f"scales{i}"] = q.scales.astype(np.float16)
        if q.zeros is not None:
            arrays[f"zeros{i}"] = q.zeros
        arrays[f"deq{i}"] = qc.dequantize(q)
        arrays[f"wire{i}"] = np.frombuffer(q.to_bytes(), np.uint8)
        meta.append(dict(c, family=fam, n=n))
    # fp16 passthrough
    i = len(meta)
    x = fam_inputs(rng, "outlier_fp16", 777) * 3
    q = qc.quantize(x, qc.PASSTHROUGH_FP16)
    arrays[f"x{i}"] = x
    arrays[f"wire{i}"] = np.frombuffer(q.to_bytes(), np.uint8)
    arrays[f"deq{i}"] = qc.dequantize(q)
    meta.append(dict(kind="fp16", family="outlier_fp16", n=777))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(out_path, **arrays)
    print(f"codec: {len(meta)} cases -> {out_path}")


# ---------------------------------------------------------------------------
# flash all-reduce with wire capture


class Capture:
    def __init__(self):
        self.msgs = {}
        self._orig = qfabric.Fabric._send

    def __enter__(self):
        cap = self

        def _send(fab, me, to, payload):
            cap.msgs.setdefault((me, to), []).append(bytes(payload))
            return cap._orig(fab, me, to, payload)

        qfabric.Fabric._send = _send
        return self

    def __exit__(self, *a):
        qfabric.Fabric._send = self._orig


def stage_codec(spec):
    if spec == "fp16":
        return qc.PASSTHROUGH_FP16
    bits, g, sym, rnd = spec
    return qc.CodecConfig(bits=bits, group_size=g, symmetric=sym, rounding=rnd)


FLASH_CASES = [
    # (n_ranks, m, stage1, stage2, chunk, family)
    (2, 4096, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), None, "gauss_bf16"),
    (4, 50000, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), None, "act"),
    (8, 65536, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), None, "act"),
    (8, 131072 + 8 * 100, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), 8 * 1024, "act"),
    (4, 40000, (8, 128, False, "nearest-even"), (8, 128, False, "nearest-even"), None, "act"),
    (4, 40000, (4, 128, False, "nearest-even"), (8, 128, False, "nearest-even"), None, "act"),  # int6
    (4, 12345, (4, 128, False, "nearest-even"), "fp16", None, "gauss_bf16"),
    (4, 3000, "fp16", "fp16", None, "int"),
    (3, 10007, (4, 32, True, "nearest-even"), (4, 32, True, "nearest-even"), None, "gauss_bf16"),
    (5, 20000, (4, 64, False, "ceil"), (4, 64, False, "ceil"), None, "gauss_bf16"),
    (4, 9000, (2, 16, False, "nearest-even"), (3, 16, False, "nearest-even"), None, "gauss_bf16"),
    (6, 7777, (5, 96, False, "nearest-even"), (7, 96, True, "nearest-even"), None, "outlier_fp16"),
    (4, 1003, (4, 64, False, "nearest-even"), (4, 64, False, "nearest-even"), None, "int"),
    (8, 8, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), None, "gauss_bf16"),
    (2, 33, (8, 2, False, "nearest-even"), (8, 2, False, "nearest-even"), None, "degenerate"),
    (4, 32768, (4, 256, False, "nearest-even"), (4, 256, False, "nearest-even"), None, "degenerate"),
    (4, 32768, (8, 32, True, "ceil"), (8, 32, False, "nearest-even"), None, "wide_exp"),
]


def rank_inputs(rng, family, n, m):
    if family == "act":
        hidden = 8192 if m % 8192 == 0 else 1000
        prof = qc.ActivationProfile(hidden_dim=hidden, tokens=-(-m // hidden), seed=int(rng.integers(1 << 30)))
        xs = qc.gen_rank_activations(prof, n)
        return [round_to_bf16(x.ravel()[:m]) for x in xs]
    if family == "int":
        return [rng.integers(-15, 16, m).astype(np.float32) for _ in range(n)]
    return [fam_inputs(rng, family, m) for _ in range(n)]


def make_flash(out_path: str) -> None:
    rng = np.random.default_rng(7)
    arrays = {}
    meta = []
    for i, (n, m, s1, s2, chunk, fam) in enumerate(FLASH_CASES):
        xs = rank_inputs(rng, fam, n, m)
        cfg = qc.FlashConfig(stage1_codec=stage_codec(s1), stage2_codec=stage_codec(s2), chunk_size=chunk)
        with Capture() as cap:
            run = qc.flash_all_reduce(xs, cfg)
        for o in run.outputs[1:]:
            assert np.array_equal(o, run.outputs[0])
        exact = qc.all_reduce_exact(xs).outputs[0]
        for r, x in enumerate(xs):
            arrays[f"c{i}_x{r}"] = x
        arrays[f"c{i}_out"] = run.outputs[0]
        arrays[f"c{i}_exact"] = exact
        for (src, dst), lst in cap.msgs.items():
            arrays[f"c{i}_w{src}_{dst}"] = np.frombuffer(b"".join(lst), np.uint8)
            arrays[f"c{i}_wlen{src}_{dst}"] = np.array([len(p) for p in lst], np.int64)
        meta.append(dict(n=n, m=m, stage1=s1, stage2=s2, chunk=chunk, family=fam,
                         wire_bytes_per_rank=run.wire_bytes_per_rank,
                         qdq=run.qdq_passes, reduce_elems=run.reduce_elems_per_rank,
                         resolved_chunk=cfg.resolve_chunk_size(n)))
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(out_path, **arrays)
    print(f"flash: {len(meta)} cases -> {out_path}")


# ---------------------------------------------------------------------------
# extras: minifloat stage codecs and the Hadamard rotation

MF_CODEC_CASES = [(fmt, g) for fmt in ("e4m3", "e5m2", "e2m1") for g in (32, 96, 128, 256)]

EXTRA_FLASH = [
    # (n_ranks, m, stage1, stage2, rotation (dim, normalize, seed) or None, family)
    (4, 40000, ("e4m3", 128), ("e4m3", 128), None, "act"),
    (8, 65536, ("e2m1", 32), ("e4m3", 32), None, "act"),
    (2, 10000, ("e5m2", 64), ("e5m2", 64), None, "gauss_bf16"),
    (4, 40960, (4, 128, False, "nearest-even"), (4, 128, False, "nearest-even"), (128, True, None), "act"),
    (8, 65536, (4, 128, False, "nearest-even"), (8, 128, False, "nearest-even"), (256, True, 3), "act"),
    (4, 12288, ("e4m3", 64), ("e4m3", 64), (64, True, 11), "gauss_bf16"),
    (2, 4096, (8, 128, True, "nearest-even"), (8, 128, True, "nearest-even"), (32, False, 5), "gauss_bf16"),
]


def extra_stage(spec):
    if isinstance(spec, tuple) and isinstance(spec[0], str):
        return qc.CodecConfig(number_format=spec[0], group_size=spec[1])
    return stage_codec(spec)


def make_extras(out_path: str) -> None:
    rng = np.random.default_rng(2412)
    arrays, mf_meta, fl_meta = {}, [], []
    for i, (fmt, g) in enumerate(MF_CODEC_CASES):
        fam = FAMILIES[i % len(FAMILIES)]
        n = int(rng.choice([997, 1024, 4096]))
        x = fam_inputs(rng, fam, n)
        cfg = qc.CodecConfig(number_format=fmt, group_size=g)
        q = qc.quantize(x, cfg)
        arrays[f"mf{i}_x"] = x
        arrays[f"mf{i}_wire"] = np.frombuffer(q.to_bytes(), np.uint8)
        arrays[f"mf{i}_deq"] = qc.dequantize(q)
        mf_meta.append(dict(format=fmt, group_size=g, family=fam, n=n))
    for i, (n, m, s1, s2, rot, fam) in enumerate(EXTRA_FLASH):
        xs = rank_inputs(rng, fam, n, m)
        rb = None if rot is None else qc.HadamardBlock(dimension=rot[0], normalize=rot[1], sign_seed=rot[2])
        cfg = qc.FlashConfig(stage1_codec=extra_stage(s1), stage2_codec=extra_stage(s2), rotation=rb)
        run = qc.flash_all_reduce(xs, cfg)
        for o in run.outputs[1:]:
            assert np.array_equal(o, run.outputs[0])
        for r, x in enumerate(xs):
            arrays[f"fl{i}_x{r}"] = x
        arrays[f"fl{i}_out"] = run.outputs[0]
        fl_meta.append(dict(n=n, m=m, stage1=s1, stage2=s2, rotation=rot, family=fam,
                            wire_bytes_per_rank=run.wire_bytes_per_rank))
    arrays["meta"] = np.frombuffer(json.dumps({"minifloat": mf_meta, "flash": fl_meta}).encode(), np.uint8)
    np.savez_compressed(out_path, **arrays)
    print(f"extras: {len(mf_meta)} minifloat codec + {len(fl_meta)} flash cases -> {out_path}")


def make_reports(out_path: str) -> None:
    rep = {"rs_vs_ag": {}, "baseline_mse": {}}
    prof = qc.ActivationProfile()
    for n in (2, 4, 8):
        for bits in (4, 8, 6):
            a, b = qc.rs_vs_ag_experiment(prof, n, bits=bits)
            rep["rs_vs_ag"][f"n{n}_b{bits}"] = [a, b]
    # 1024x8192 outlier activations cast to bf16, flash vs exact
    for n in (2, 4, 8):
        xs = qc.gen_rank_activations(qc.ActivationProfile(hidden_dim=8192, tokens=1024, seed=0), n)
        xs = [round_to_bf16(x) for x in xs]
        exact = qc.all_reduce_exact(xs).outputs[0]
        for bits in (8, 6, 4):
            out = qc.flash_all_reduce(xs, qc.FlashConfig.from_bits(bits)).outputs[0]
            rep["baseline_mse"][f"n{n}_b{bits}"] = qc.mse(out, exact)
            print("baseline mse", n, bits, rep["baseline_mse"][f"n{n}_b{bits}"], flush=True)
    with open(out_path, "w") as fh:
        json.dump(rep, fh, indent=1, sort_keys=True)
    print(f"reports -> {out_path}")


# ---------------------------------------------------------------------------
# full-size digests: the unmodified reference at the BASELINE configs

DIGEST_CASES = [
    # (name, n_ranks, tokens, hidden, bits preset, input dtype)
    ("c1_tp4_int8_fp16", 4, 1024, 8192, 8, "fp16"),
    ("tp8_int8_bf16", 8, 1024, 8192, 8, "bf16"),
    ("tp8_int6_bf16", 8, 1024, 8192, 6, "bf16"),
    ("c2_tp8_int4_bf16", 8, 8192, 8192, 4, "bf16"),
]


def _sha(b) -> str:
    import hashlib

    return hashlib.sha256(bytes(memoryview(np.ascontiguousarray(b)).cast("B")) if not isinstance(b, bytes) else b).hexdigest()


def split_wire(msgs, plen, codec):
    """codes / scales / zeros parts of a list of per-piece wire messages, each concatenated."""
    from qcollectives.bitpack import packed_byte_len

    packed = packed_byte_len(plen, codec.storage_bits)
    groups = codec.group_count(plen)
    codes, scales, zeros = [], [], []
    for m in msgs:
        codes.append(m[:packed])
        scales.append(m[packed:packed + 2 * groups])
        zeros.append(m[packed + 2 * groups:])
    return b"".join(codes), b"".join(scales), b"".join(zeros)


def make_digests(out_path: str, only=None) -> None:
    import time

    res = {}
    if os.path.exists(out_path):
        with open(out_path) as fh:
            res = json.load(fh)
    for name, n, tokens, hidden, bits, dt in DIGEST_CASES:
        if only and name not in only:
            continue
        t0 = time.time()
        prof = qc.ActivationProfile(hidden_dim=hidden, tokens=tokens, seed=0)
        xs = qc.gen_rank_activations(prof, n)
        rnd = round_to_bf16 if dt == "bf16" else round_to_fp16
        xs = [rnd(x) for x in xs]
        cfg = qc.FlashConfig.from_bits(bits)
        with Capture() as cap:
            run = qc.flash_all_reduce(xs, cfg)
        for o in run.outputs[1:]:
            assert np.array_equal(o, run.outputs[0])
        m = xs[0].size
        seg = m // n
        plen = cfg.resolve_chunk_size(n) // n
        s1, s2 = cfg.stage1_codec, cfg.stage2_codec
        d = {"n": n, "m": m, "tokens": tokens, "hidden": hidden, "bits": bits, "dtype": dt, "seed": 0,
             "piece": plen, "inputs": [_sha(x.astype(np.float32)) for x in xs],
             "out_f32": _sha(run.outputs[0].astype(np.float32)), "stage1": {}, "stage2": {},
             "wire_bytes_per_rank": run.wire_bytes_per_rank}
        for (src, dst), lst in sorted(cap.msgs.items()):
            # per (src, dst) and piece: one stage-1 message, then one stage-2 message (collectives.py:359-381)
            assert len(lst) == 2 * (seg // plen)
            c, sc, z = split_wire(lst[0::2], plen, s1)
            d["stage1"][f"{src}->{dst}"] = [_sha(c), _sha(sc), _sha(z)]
            c, sc, z = split_wire(lst[1::2], plen, s2)
            key = str(src)
            dig = [_sha(c), _sha(sc), _sha(z)]
            assert d["stage2"].setdefault(key, dig) == dig  # the owner sends one payload to every peer
        res[name] = d
        print(f"digest {name}: {time.time() - t0:.1f} s", flush=True)
        del run, xs, cap
        with open(out_path, "w") as fh:
            json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["codec", "flash", "reports", "extras", "digests"]
    if "codec" in which:
        make_codec(os.path.join(HERE, "codec.npz"))
    if "flash" in which:
        make_flash(os.path.join(HERE, "flash.npz"))
    if "reports" in which:
        make_reports(os.path.join(HERE, "reports.json"))
    if "extras" in which:
        make_extras(os.path.join(HERE, "extras.npz"))
    if "digests" in which:
        make_digests(os.path.join(HERE, "digests.json"), [w for w in which if w != "digests"])
