"""Caller integration: the flash all-reduce as the reduction of a tensor-parallel
row-linear layer (arXiv 2412.04964 §3, PAPER.md:133 — o_proj / down_proj).

* `torch.ops.flashcomm.all_reduce_(x, bits, group_size, symmetric)` — a
  `torch.library` custom op, in place on the GEMM output, stream-ordered and
  host-sync free, so it can be captured in a CUDA graph (the communicator's
  peer buffers are fixed at creation; every call advances the epoch flags).
* `FlashRowParallelLinear` — y = x_shard @ W_shard^T, flash all-reduced in
  place across the TP group, + bias.

One process per GPU: `set_comm(FlashComm.from_process_group(...))` once per
process (the reference's `flash_all_reduce` call, collectives.py:321, with the
TP group's world size).
"""

from __future__ import annotations

from typing import Optional

import torch

from .codec import CodecConfig
from .collectives import FlashConfig
from .comm import FlashComm
from .errors import ConfigError

_COMM: dict = {}


def set_comm(comm: FlashComm, device: Optional[int] = None) -> None:
    """Register the per-rank communicator used by the op on `device`."""
    if comm.rank is None:
        raise ConfigError("the TP op needs a per-rank (IPC) communicator: FlashComm.from_process_group")
    _COMM[int(device if device is not None else comm.devices[comm.rank])] = comm


def get_comm(device: int) -> FlashComm:
    comm = _COMM.get(int(device))
    if comm is None:
        raise ConfigError(f"no flash communicator registered for cuda:{device} (call paper_2412_04964_b200.tp.set_comm)")
    return comm


def clear_comms() -> None:
    _COMM.clear()


def _config(bits: int, group_size: int, symmetric: bool) -> FlashConfig:
    if bits == 6 and not symmetric:
        return FlashConfig.int6(group_size=group_size)
    if bits in (16,):
        return FlashConfig.from_bits(16)
    return FlashConfig.uniform(CodecConfig(bits=bits, group_size=group_size, symmetric=symmetric))


@torch.library.custom_op("flashcomm::all_reduce_", mutates_args=("x",))
def all_reduce_(x: torch.Tensor, bits: int, group_size: int, symmetric: bool) -> None:
    """In-place flash all-reduce of a contiguous CUDA tensor across the TP group."""
    comm = get_comm(x.device.index)
    comm.all_reduce(x, _config(bits, group_size, symmetric), out=x, check=False)


@all_reduce_.register_fake
def _(x, bits, group_size, symmetric):  # noqa: ANN001
    return None


class FlashRowParallelLinear(torch.nn.Module):
    """Row-parallel linear: this rank holds in_features/tp input columns of the
    weight; the partial products are summed with the flash all-reduce."""

    def __init__(self, in_features_per_rank: int, out_features: int, bits: int = 4, group_size: int = 128,
                 symmetric: bool = False, bias: bool = False, device=None, dtype=torch.bfloat16):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features_per_rank, device=device, dtype=dtype))
        self.bias = torch.nn.Parameter(torch.zeros(out_features, device=device, dtype=dtype)) if bias else None
        self.bits, self.group_size, self.symmetric = int(bits), int(group_size), bool(symmetric)
        torch.nn.init.normal_(self.weight, std=in_features_per_rank ** -0.5)

    def forward(self, x_shard: torch.Tensor) -> torch.Tensor:
        y = torch.matmul(x_shard, self.weight.t()).contiguous()
        torch.ops.flashcomm.all_reduce_(y, self.bits, self.group_size, self.symmetric)
        if self.bias is not None:
            y = y + self.bias
        return y
