"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 Flash All-Reduce. It restates,
in vectorised numpy float64 arithmetic, the reference algorithm of
arXiv 2412.04964's `qcollectives` package (read-only at /root/reference/pkg).
Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it. The product package
(`paper_2412_04964_b200`) never imports, links or executes anything here; its
compute path is the sm_100a CUDA library and fails loudly without it.

Parity pins: this restatement is checked against golden vectors produced by
the reference itself (`tests/golden/make_golden.py` -> `tests/golden/*.npz`,
including the reference's own wire messages captured from its fabric) and
against the known-answer tests of the reference test-suite
(`tests/test_oracle_golden.py`).

Restatement choices
-------------------
* Segment form of Alg. 1. The reference quantizes per piece of each rank
  segment (collectives.py:359-367); pieces are multiples of every quantizing
  group size (collectives.py:65-75) and groups are anchored at the piece start,
  so quantizing a whole segment at once yields identical groups, codes and
  sums (collectives.py:14-16; reference test test_collectives.py:164-174).
* Float64 parameter math exactly as numpy does it in the reference
  (codec.py:292-329): min/max/absmax in f64, scale division in f64, one
  f64->f16 rounding, ceil/round in f64.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

FP16_MAX = 65504.0
DEFAULT_CHUNK_ELEMS = 64 * 1024  # collectives.py:32


# --------------------------------------------------------------------------
# minifloat formats (restated from minifloat.py:22-124): sign / exponent /
# mantissa with IEEE-style subnormals, round-to-nearest-even, saturating at
# the largest finite magnitude (no inf/NaN patterns are produced)


@dataclass(frozen=True)
class MiniFloat:
    name: str
    exp_bits: int
    mantissa_bits: int
    bias: int
    max_finite: float

    @property
    def code_bits(self) -> int:
        return 1 + self.exp_bits + self.mantissa_bits

    @property
    def min_normal(self) -> float:
        return 2.0 ** (1 - self.bias)

    @property
    def sub_quantum(self) -> float:
        return 2.0 ** (1 - self.bias - self.mantissa_bits)


MINIFLOATS = {f.name: f for f in (MiniFloat("e4m3", 4, 3, 7, 448.0), MiniFloat("e5m2", 5, 2, 15, 57344.0),
                                  MiniFloat("e2m1", 2, 1, 1, 6.0))}


def mf_round(x: np.ndarray, f: MiniFloat) -> np.ndarray:
    """minifloat.py:58-76: nearest grid value (float64), ties to even, saturating."""
    x = np.asarray(x, np.float64)
    a = np.abs(x)
    _, e2 = np.frexp(a)
    quantum = np.where(a < f.min_normal, f.sub_quantum, np.exp2(e2 - 1 - f.mantissa_bits))
    r = np.minimum(np.round(a / quantum) * quantum, f.max_finite)
    return np.where(x < 0, -r, r)


def mf_encode(v: np.ndarray, f: MiniFloat) -> np.ndarray:
    """minifloat.py:79-100: grid values -> uint8 bit patterns."""
    v = np.asarray(v, np.float64)
    sign = (v < 0).astype(np.int64)
    a = np.abs(v)
    sub = a < f.min_normal
    _, e2 = np.frexp(a)
    e = e2 - 1
    expc = np.where(sub, 0, e + f.bias).astype(np.int64)
    mant = np.where(sub, a / f.sub_quantum, (a * np.exp2(-e) - 1.0) * (1 << f.mantissa_bits))
    code = (sign << (f.exp_bits + f.mantissa_bits)) | (expc << f.mantissa_bits) | np.round(mant).astype(np.int64)
    return code.astype(np.uint8)


def mf_table(f: MiniFloat) -> np.ndarray:
    """minifloat.py:103-118: float32 value of every code pattern."""
    out = np.empty(1 << f.code_bits, np.float32)
    for code in range(out.size):
        sgn = -1.0 if code >> (f.exp_bits + f.mantissa_bits) else 1.0
        ec = (code >> f.mantissa_bits) & ((1 << f.exp_bits) - 1)
        mc = code & ((1 << f.mantissa_bits) - 1)
        mag = mc * f.sub_quantum if ec == 0 else (1 + mc / (1 << f.mantissa_bits)) * 2.0 ** (ec - f.bias)
        out[code] = np.float32(sgn * mag)
    return out


# --------------------------------------------------------------------------
# Hadamard rotation (restated from rotation.py:21-83)


@dataclass(frozen=True)
class Hadamard:
    dimension: int
    normalize: bool = True
    sign_seed: Optional[int] = None

    def signs(self) -> Optional[np.ndarray]:
        if self.sign_seed is None:
            return None
        return np.random.default_rng(self.sign_seed).choice(np.array([-1.0, 1.0]), size=self.dimension)


def _fwht(blocks: np.ndarray) -> np.ndarray:
    rows, dim = blocks.shape
    y, h = blocks, 1
    while h < dim:
        y = y.reshape(rows, dim // (2 * h), 2, h)
        y = np.stack([y[:, :, 0, :] + y[:, :, 1, :], y[:, :, 0, :] - y[:, :, 1, :]], axis=2).reshape(rows, dim)
        h *= 2
    return y


def hadamard_apply(x: np.ndarray, hb: Hadamard) -> np.ndarray:
    """rotation.py:61-71: H(D x) per block of `dimension`, float64, one cast to float32."""
    b = np.asarray(x, np.float64).ravel().reshape(-1, hb.dimension).copy()
    sg = hb.signs()
    if sg is not None:
        b *= sg
    y = _fwht(b)
    if hb.normalize:
        y = y / np.sqrt(hb.dimension)
    return y.ravel().astype(np.float32)


def hadamard_inverse(x: np.ndarray, hb: Hadamard) -> np.ndarray:
    """rotation.py:74-83: D(H x) / sqrt(dim) (normalized) or / dim."""
    y = _fwht(np.asarray(x, np.float64).ravel().reshape(-1, hb.dimension).copy())
    y = y / np.sqrt(hb.dimension) if hb.normalize else y / hb.dimension
    sg = hb.signs()
    if sg is not None:
        y *= sg
    return y.ravel().astype(np.float32)


# --------------------------------------------------------------------------
# codec descriptor (mirror of codec.py:45-133, restated)


@dataclass(frozen=True)
class Codec:
    """kind: 'int' (bits 2..8), 'fp16' (passthrough) or a minifloat format
    'e4m3' / 'e5m2' / 'e2m1' (group-scaled, codec.py:332-351)."""

    kind: str = "int"
    bits: int = 4
    group_size: int = 128
    symmetric: bool = False
    rounding: str = "nearest-even"
    scale_floor: float = 1e-8

    @property
    def storage_bits(self) -> int:  # codec.py:98-103
        if self.kind == "fp16":
            return 16
        if self.kind in MINIFLOATS:
            return 4 if MINIFLOATS[self.kind].code_bits <= 4 else 8
        return 4 if self.bits <= 4 else 8

    @property
    def meta_bytes(self) -> int:  # codec.py:105-112
        if self.kind == "fp16":
            return 0
        return 2 if (self.symmetric or self.kind != "int") else 3

    def groups(self, n: int) -> int:  # codec.py:123-126
        return 0 if self.kind == "fp16" else -(-n // self.group_size)

    def wire_len(self, n: int) -> int:  # codec.py:128-133
        if self.kind == "fp16":
            return 2 * n
        return packed_len(n, self.storage_bits) + self.groups(n) * self.meta_bytes


FP16 = Codec(kind="fp16")


def packed_len(n: int, bits: int) -> int:  # bitpack.py:20-24
    return (n * bits + 7) // 8


# --------------------------------------------------------------------------
# bit packing (bitpack.py:48-75): little-nibble-first


def pack(codes: np.ndarray, bits: int) -> np.ndarray:
    c = np.ascontiguousarray(codes, dtype=np.uint8).ravel()
    if bits == 8:
        return c.copy()
    if c.size % 2:
        c = np.concatenate([c, np.zeros(1, np.uint8)])
    return (c[0::2] | (c[1::2] << 4)).astype(np.uint8)


def unpack(data: np.ndarray, n: int, bits: int) -> np.ndarray:
    d = np.asarray(data, dtype=np.uint8).ravel()
    if bits == 8:
        return d[:n].copy()
    out = np.empty(d.size * 2, np.uint8)
    out[0::2] = d & 0x0F
    out[1::2] = d >> 4
    return out[:n]


# --------------------------------------------------------------------------
# group codec


def _group_starts(n: int, g: int) -> np.ndarray:
    return np.arange(0, n, g)


def _expand(per_group: np.ndarray, n: int, g: int) -> np.ndarray:
    # broadcast one value per group back over its elements; last group may be short
    return np.repeat(per_group, g)[:n]


def snap_scale_f16(raw: np.ndarray, floor: float) -> np.ndarray:
    """f64 raw scale -> fp16 wire scale (codec.py:235-248).

    max(raw, floor); one RNE rounding to fp16; overflow clamps to 65504; a
    result below the floor (incl. underflow to 0) moves one fp16 ulp up.
    """
    r = np.maximum(np.asarray(raw, np.float64), floor)
    h = r.astype(np.float16)
    h = np.where(np.isinf(h), np.float16(FP16_MAX), h)
    bump = h.astype(np.float64) < floor
    if bump.any():
        h = np.where(bump, np.nextafter(h, np.float16(np.inf)), h)
    return h.astype(np.float16)


def _round(v: np.ndarray, mode: str) -> np.ndarray:  # codec.py:288-289
    return np.round(v) if mode == "nearest-even" else np.ceil(v)


@dataclass
class QSeg:
    """Quantized segment: unpacked codes (uint8 per element, two's complement
    low bits for symmetric), fp16 scales, uint8 zeros (asym int only)."""

    codes: np.ndarray
    scales: np.ndarray
    zeros: Optional[np.ndarray]
    n: int
    codec: Codec

    def wire_bytes(self) -> bytes:
        """codes || fp16 scales || zeros (codec.py:193-200)."""
        if self.codec.kind == "fp16":
            return self.codes.tobytes()
        parts = [pack(self.codes, self.codec.storage_bits).tobytes(), self.scales.astype(np.float16).tobytes()]
        if self.zeros is not None:
            parts.append(self.zeros.astype(np.uint8).tobytes())
        return b"".join(parts)


def quantize(x, codec: Codec) -> QSeg:
    """Group quantizer restated from codec.py:292-329 (int) / :294-298 (fp16).

    For the fp16 passthrough `codes` holds the raw little-endian fp16 bytes.
    """
    a = np.asarray(x, dtype=np.float64).ravel()
    if a.size == 0:
        raise ValueError("empty input")  # codec.py:228-229 (DomainError)
    if not np.isfinite(a).all():
        raise ValueError("non-finite input")  # codec.py:230-231 (DomainError)
    n = a.size
    if codec.kind == "fp16":
        return QSeg(a.astype(np.float16).view(np.uint8).copy(), np.empty(0, np.float16), None, n, codec)
    if codec.kind in MINIFLOATS:  # codec.py:332-351: absmax / max_finite scale, grid rounding, saturating
        f = MINIFLOATS[codec.kind]
        amax = np.maximum.reduceat(np.abs(a), _group_starts(n, codec.group_size))
        s16 = snap_scale_f16(amax / f.max_finite, codec.scale_floor)
        se = _expand(s16.astype(np.float64), n, codec.group_size)
        return QSeg(mf_encode(mf_round(a / se, f), f), s16, None, n, codec)
    g, b = codec.group_size, codec.bits
    st = _group_starts(n, g)
    if codec.symmetric:
        amax = np.maximum.reduceat(np.abs(a), st)
        s16 = snap_scale_f16(amax / (2 ** (b - 1) - 1), codec.scale_floor)
        se = _expand(s16.astype(np.float64), n, g)
        q = np.clip(_round(a / se, codec.rounding), -(2 ** (b - 1)), 2 ** (b - 1) - 1).astype(np.int64)
        codes = (q & ((1 << b) - 1)).astype(np.uint8)
        return QSeg(codes, s16, None, n, codec)
    lo = np.minimum.reduceat(a, st)
    hi = np.maximum.reduceat(a, st)
    qmax = 2 ** b - 1
    s16 = snap_scale_f16((hi - lo) / qmax, codec.scale_floor)
    s = s16.astype(np.float64)
    z = np.clip(np.ceil(-lo / s), 0, qmax).astype(np.int64)
    q = np.clip(_round(a / _expand(s, n, g), codec.rounding) + _expand(z, n, g), 0, qmax)
    return QSeg(q.astype(np.uint8), s16, z.astype(np.uint8), n, codec)


def dequantize(q: QSeg) -> np.ndarray:
    """Restated from codec.py:354-384: (c - z) * s, or sign-extended c * s."""
    c = q.codec
    if c.kind == "fp16":
        return q.codes.view(np.float16).astype(np.float32)
    n, g = q.n, c.group_size
    se = _expand(q.scales.astype(np.float64), n, g)
    if c.kind in MINIFLOATS:  # codec.py:376-379
        return (mf_table(MINIFLOATS[c.kind])[q.codes].astype(np.float64) * se).astype(np.float32)
    v = q.codes.astype(np.int64)
    if c.symmetric:
        v = v - ((v >> (c.bits - 1)) & 1) * (1 << c.bits)
        return (v * se).astype(np.float32)
    return ((v - _expand(q.zeros.astype(np.int64), n, g)) * se).astype(np.float32)


def mse(a, b) -> float:  # codec.py:387-393
    x = np.asarray(a, np.float64).ravel()
    y = np.asarray(b, np.float64).ravel()
    return float(np.mean((x - y) ** 2))


# --------------------------------------------------------------------------
# collectives


def resolve_chunk(n_ranks: int, stage1: Codec, stage2: Codec, chunk: Optional[int] = None) -> int:
    """collectives.py:56-75."""
    mult = 1
    for c in (stage1, stage2):
        if c.kind != "fp16":
            mult = math.lcm(mult, c.group_size)
    unit = n_ranks * mult
    if chunk is None:
        return max(1, math.ceil(DEFAULT_CHUNK_ELEMS / unit)) * unit
    if chunk % unit:
        raise ValueError(f"chunk {chunk} not a multiple of {unit}")
    return chunk


def _padded(flat: np.ndarray, n_ranks: int) -> tuple[np.ndarray, int]:
    """collectives.py:145-149: zero-pad to N equal segments."""
    seg = -(-flat.size // n_ranks)
    p = np.zeros(n_ranks * seg, np.float32)
    p[: flat.size] = flat
    return p, seg


def sequential_sum(parts: Sequence[np.ndarray]) -> np.ndarray:
    """collectives.py:182-187: float32, ascending rank order."""
    acc = np.array(parts[0], np.float32, copy=True)
    for p in parts[1:]:
        acc += np.asarray(p, np.float32)
    return acc


@dataclass
class FlashResult:
    outputs: list  # float32, original shape, one per rank (identical)
    stage1: list  # stage1[j][s]: QSeg of source s's segment j
    stage2: list  # stage2[j]: QSeg of reduced segment j
    reduced: list  # fp32 sums per segment (pre stage-2)
    seg: int
    wire_bytes_per_rank: int


def flash_all_reduce(tensors: Sequence[np.ndarray], stage1: Codec, stage2: Codec,
                     chunk: Optional[int] = None, rotation: Optional[Hadamard] = None) -> FlashResult:
    """Segment restatement of flash_all_reduce (collectives.py:321-402); with
    `rotation` the padded rank tensors are Hadamard-rotated before and the
    outputs rotated back after (collectives.py:350-351,390-391)."""
    flats = [np.asarray(t, np.float32).ravel() for t in tensors]
    n = len(flats)
    shape = np.asarray(tensors[0]).shape
    m = flats[0].size
    if n == 1:
        return FlashResult([flats[0].reshape(shape).copy()], [], [], [], m, 0)
    piece = resolve_chunk(n, stage1, stage2, chunk) // n
    padded = [_padded(f, n)[0] for f in flats]
    if rotation is not None:
        padded = [hadamard_apply(p, rotation) for p in padded]
    seg = padded[0].size // n
    st1 = [[quantize(padded[s][j * seg:(j + 1) * seg], stage1) for s in range(n)] for j in range(n)]
    reduced = [sequential_sum([dequantize(q) for q in st1[j]]) for j in range(n)]
    st2 = [quantize(r, stage2) for r in reduced]
    out = np.concatenate([dequantize(q) for q in st2])
    if rotation is not None:
        out = hadamard_inverse(out, rotation)
    out = out[:m].reshape(shape)
    # wire accounting (costmodel.py:122-128 == fabric ledger of rank 0)
    wire = 0
    off = 0
    while off < seg:
        plen = min(piece, seg - off)
        wire += stage1.wire_len(plen) + stage2.wire_len(plen)
        off += piece
    return FlashResult([out.copy() for _ in range(n)], st1, st2, reduced, seg, (n - 1) * wire)


def piece_messages(q: QSeg, piece: int) -> list[bytes]:
    """Split a segment's quantization into the reference's per-piece wire
    messages (collectives.py:152-157,363,377): valid because piece % g == 0."""
    out = []
    c = q.codec
    for off in range(0, q.n, piece):
        plen = min(piece, q.n - off)
        if c.kind == "fp16":
            out.append(q.codes[2 * off: 2 * (off + plen)].tobytes())
            continue
        g0, g1 = off // c.group_size, -(-(off + plen) // c.group_size)
        sub = QSeg(q.codes[off:off + plen], q.scales[g0:g1],
                   None if q.zeros is None else q.zeros[g0:g1], plen, c)
        out.append(sub.wire_bytes())
    return out


def all_reduce_exact(tensors: Sequence[np.ndarray]) -> np.ndarray:
    """collectives.py:190-241: fp32 rank-ordered sum, returned once."""
    flats = [np.asarray(t, np.float32).ravel() for t in tensors]
    shape = np.asarray(tensors[0]).shape
    return sequential_sum(flats).reshape(shape)


# --------------------------------------------------------------------------
# synthetic activations (workload.py:34-120, restated)


def gen_activations(hidden: int, tokens: int, seed, base_std: float = 1.0,
                    outlier_frac: float = 0.01, outlier_scale: float = 30.0,
                    placement: str = "scattered") -> np.ndarray:
    rng = np.random.default_rng(seed)
    k = int(round(outlier_frac * hidden))
    if k == 0:
        ch = np.empty(0, np.int64)
    elif placement == "banded":
        start = int(rng.integers(0, hidden - k + 1))
        ch = np.arange(start, start + k)
    else:
        ch = rng.choice(hidden, size=k, replace=False)
    x = rng.standard_normal((tokens, hidden)) * base_std
    if ch.size:
        x[:, ch] *= outlier_scale
    return x.astype(np.float32)


def gen_rank_activations(hidden: int, tokens: int, seed: int, n_ranks: int, **kw) -> list:
    kids = np.random.SeedSequence(seed).spawn(n_ranks)
    return [gen_activations(hidden, tokens, k, **kw) for k in kids]


# --------------------------------------------------------------------------
# bf16 helpers (numpy has no bfloat16)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bit patterns (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(f32_to_bf16_bits(x)).reshape(np.shape(x))


def round_to_fp16(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)
