"""Canonical code packing (the reference's `qcollectives.bitpack`,
/root/reference/pkg/src/qcollectives/bitpack.py:20-89) on torch tensors.

The kernels pack in registers (little-nibble-first INT4, bytes for 5..8
bits); these thin entry points expose the same layout for callers and tests
that hold unpacked codes: `pack(codes, bits)` / `unpack(buf, count, bits)` /
`packed_byte_len` / `magic_dequant_identity`, with the reference's errors.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import DomainError, IntegrityError

SUPPORTED_WIDTHS = (4, 8)


def packed_byte_len(code_count: int, bits_per_code: int) -> int:
    """Bytes for `code_count` codes of `bits_per_code` bits (bitpack.py:20-24)."""
    if bits_per_code not in SUPPORTED_WIDTHS:
        raise DomainError(f"bits must be one of {SUPPORTED_WIDTHS}, got {bits_per_code}")
    return (int(code_count) * bits_per_code + 7) // 8


def pack(codes, bits: int) -> torch.Tensor:
    """Pack unsigned codes (any integer tensor/array) into a uint8 tensor on the
    codes' device: INT4 code i in the low nibble of byte i//2 when i is even,
    the high nibble when odd (bitpack.py:48-62); odd counts pad a 0 nibble."""
    if bits not in SUPPORTED_WIDTHS:
        raise DomainError(f"bits must be one of {SUPPORTED_WIDTHS}, got {bits}")
    t = codes if isinstance(codes, torch.Tensor) else torch.as_tensor(np.asarray(codes))
    t = t.reshape(-1)
    if t.numel() and (int(t.min()) < 0 or int(t.max()) >= (1 << bits)):
        raise DomainError(f"codes out of range for {bits}-bit packing")
    t = t.to(torch.uint8)
    if bits == 8:
        return t.clone()
    if t.numel() % 2:
        t = torch.cat([t, t.new_zeros(1)])
    return (t[0::2] | (t[1::2] << 4)).contiguous()


def unpack(buf: torch.Tensor, code_count: int, bits: int) -> torch.Tensor:
    """Exact inverse of pack (bitpack.py:64-75)."""
    if bits not in SUPPORTED_WIDTHS:
        raise DomainError(f"bits must be one of {SUPPORTED_WIDTHS}, got {bits}")
    raw = buf.reshape(-1).to(torch.uint8)
    if raw.numel() != packed_byte_len(code_count, bits):
        raise IntegrityError(f"buffer holds {raw.numel()} bytes, expected {packed_byte_len(code_count, bits)} "
                             f"for {code_count} codes of {bits} bits")
    if bits == 8:
        return raw.clone()
    out = torch.stack([raw & 0x0F, raw >> 4], dim=1).reshape(-1)
    return out[:code_count].contiguous()


def magic_dequant_identity(code: int) -> float:
    """fp16 exponent-bias decode of a 4-bit code: 0x6400 | code is 1024 + code
    (bitpack.py:78-89); the kernels use the fp32 form (2^23 + c, PRMT)."""
    if not 0 <= int(code) <= 15:
        raise DomainError(f"code must be in 0..15, got {code}")
    return float(np.uint16(0x6400 | int(code)).view(np.float16)) - 1024.0
