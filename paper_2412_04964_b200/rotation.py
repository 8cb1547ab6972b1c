"""Blocked Hadamard rotation for outlier spreading (the reference's
rotation.py:21-83, the §5.2 ablation), on the GPU: `fc_hadamard` runs the
butterflies in float64 in the reference's order, so results are bit-identical
to the reference's numpy transform."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .codec import fc_dtype
from .errors import ConfigError


@dataclass(frozen=True)
class HadamardBlock:
    """rotation.py:21-35: block dimension (power of two), orthonormal scaling,
    optional seeded random sign diagonal."""

    dimension: int
    normalize: bool = True
    sign_seed: Optional[int] = None

    def __post_init__(self) -> None:
        d = int(self.dimension)
        if d < 1 or (d & (d - 1)) != 0:
            raise ConfigError(f"dimension must be a power of two >= 1, got {self.dimension}")

    def signs(self) -> Optional[np.ndarray]:
        if self.sign_seed is None:
            return None
        rng = np.random.default_rng(self.sign_seed)
        return rng.choice(np.array([-1.0, 1.0]), size=self.dimension)

    def _device_signs(self, device: torch.device) -> Optional[torch.Tensor]:
        s = self.signs()
        return None if s is None else torch.from_numpy(s.astype(np.float32)).to(device)


def _run(x: torch.Tensor, block: HadamardBlock, n_padded: int, inverse: bool, out_dtype: torch.dtype,
         n_out: int) -> torch.Tensor:
    if not x.is_cuda or not x.is_contiguous():
        raise ConfigError("Hadamard rotation needs a contiguous CUDA tensor")
    out = torch.empty(n_out, dtype=out_dtype, device=x.device)
    signs = block._device_signs(x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().fc_hadamard(x.data_ptr(), fc_dtype(x.dtype), x.numel(), int(n_padded),
                                          int(block.dimension), int(bool(block.normalize)),
                                          signs.data_ptr() if signs is not None else None, int(inverse),
                                          out.data_ptr(), fc_dtype(out_dtype), int(n_out),
                                          torch.cuda.current_stream(x.device).cuda_stream))
    return out


def hadamard_apply(x: torch.Tensor, block: HadamardBlock, n_padded: Optional[int] = None) -> torch.Tensor:
    """rotation.py:61-71: float32 H(D x) of the (zero-padded to n_padded) flat tensor."""
    x = x.reshape(-1)
    n_padded = x.numel() if n_padded is None else int(n_padded)
    return _run(x, block, n_padded, False, torch.float32, n_padded)


def hadamard_inverse(x: torch.Tensor, block: HadamardBlock, out_dtype: torch.dtype = torch.float32,
                     n_out: Optional[int] = None) -> torch.Tensor:
    """rotation.py:74-83: the exact inverse; the first n_out elements in out_dtype."""
    x = x.reshape(-1)
    return _run(x, block, x.numel(), True, out_dtype, x.numel() if n_out is None else int(n_out))
