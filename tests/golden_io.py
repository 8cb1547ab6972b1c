"""Loaders for the committed golden fixtures (made by tests/golden/make_golden.py
from the unmodified reference implementation)."""

from __future__ import annotations

import json
import os
from functools import lru_cache

import numpy as np

from oracle import flash_oracle as orc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@lru_cache(maxsize=None)
def codec_npz():
    return np.load(os.path.join(GOLDEN, "codec.npz"))


@lru_cache(maxsize=None)
def flash_npz():
    return np.load(os.path.join(GOLDEN, "flash.npz"))


def codec_meta():
    return json.loads(bytes(codec_npz()["meta"]).decode())


def flash_meta():
    return json.loads(bytes(flash_npz()["meta"]).decode())


def reports():
    with open(os.path.join(GOLDEN, "reports.json")) as fh:
        return json.load(fh)


def oracle_codec(meta: dict) -> orc.Codec:
    if meta.get("kind") == "fp16":
        return orc.FP16
    return orc.Codec(bits=meta["bits"], group_size=meta["group_size"],
                     symmetric=meta["symmetric"], rounding=meta["rounding"])


def oracle_stage(spec) -> orc.Codec:
    if spec == "fp16":
        return orc.FP16
    bits, g, sym, rnd = spec
    return orc.Codec(bits=bits, group_size=g, symmetric=sym, rounding=rnd)


def flash_case(i: int):
    z = flash_npz()
    m = flash_meta()[i]
    xs = [z[f"c{i}_x{r}"] for r in range(m["n"])]
    return m, xs, z[f"c{i}_out"], z[f"c{i}_exact"]


def flash_wire(i: int, src: int, dst: int) -> list[bytes]:
    z = flash_npz()
    blob = bytes(z[f"c{i}_w{src}_{dst}"])
    lens = z[f"c{i}_wlen{src}_{dst}"]
    out, off = [], 0
    for ln in lens:
        out.append(blob[off:off + int(ln)])
        off += int(ln)
    return out


@lru_cache(maxsize=None)
def extras_npz():
    return np.load(os.path.join(GOLDEN, "extras.npz"))


def extras_meta():
    return json.loads(bytes(extras_npz()["meta"]).decode())


def extra_stage(spec) -> orc.Codec:
    """Stage spec of extras.npz: [format, group] for minifloats, else oracle_stage."""
    if isinstance(spec, (list, tuple)) and isinstance(spec[0], str):
        return orc.Codec(kind=spec[0], group_size=spec[1])
    return oracle_stage(spec)
