"""Flash All-Reduce on B200: the reference's `qcollectives.collectives`
interface (/root/reference/pkg/src/qcollectives/collectives.py) over CUDA
tensors.

`flash_all_reduce(tensors, cfg, topology=None, timeout=5.0)` keeps the
reference signature (collectives.py:321-326): one tensor per rank. The ranks
may be several GPUs of this process (P2P over NVLink) or several logical
ranks sharing one GPU; either way the work runs in libflashcomm's sm_100a
kernels (stage-1 quantize fused with the all-to-all stores into peer
buffers; dequantize + fp32 sum + requantize + broadcast; gather-dequantize).
For one process per GPU (torchrun), use `FlashComm.from_process_group` and
`FlashComm.all_reduce`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from .codec import CodecConfig, PASSTHROUGH_FP16, as_device_tensor, as_host_tensor, int6_flash_pair
from .comm import DEFAULT_TIMEOUT_S, FabricTopology, FlashComm, TrafficLedger, flash_ledger, slot_bytes_for
from .errors import ConfigError, DomainError, ProtocolError

DEFAULT_CHUNK_ELEMS = 64 * 1024  # collectives.py:32
METHODS = ("exact", "ring", "flash")


@dataclass(frozen=True)
class FlashConfig:
    """Stage codecs and blocking of the two-step quantized all-reduce
    (collectives.py:37-109). `chunk_size` is validated like the reference but
    never changes results (collectives.py:14-16). `rotation` (rotation.HadamardBlock,
    rotation.py) is fused into the lane-8 kernels when its block (<= 256) tiles the
    rank segments, else applied as separate passes around the all-reduce."""

    stage1_codec: CodecConfig
    stage2_codec: CodecConfig
    chunk_size: Optional[int] = None
    rotation: Optional[object] = None

    def __post_init__(self) -> None:
        if self.chunk_size is not None and self.chunk_size < 1:
            raise ConfigError(f"chunk_size must be positive, got {self.chunk_size}")

    @property
    def group_multiple(self) -> int:
        mult = 1
        for c in (self.stage1_codec, self.stage2_codec):
            if not c.is_passthrough:
                mult = math.lcm(mult, c.group_size)
        return mult

    def resolve_chunk_size(self, world_size: int) -> int:  # collectives.py:65-75
        unit = world_size * self.group_multiple
        if self.chunk_size is None:
            return max(1, math.ceil(DEFAULT_CHUNK_ELEMS / unit)) * unit
        if self.chunk_size % unit:
            raise ConfigError(f"chunk_size {self.chunk_size} must be a multiple of world_size*group lcm = {unit}")
        return self.chunk_size

    def to_json_dict(self) -> dict:
        return {"stage1": self.stage1_codec.to_json_dict(), "stage2": self.stage2_codec.to_json_dict(),
                "chunk_size": self.chunk_size}

    @classmethod
    def uniform(cls, codec: CodecConfig, **kw) -> "FlashConfig":
        return cls(stage1_codec=codec, stage2_codec=codec, **kw)

    @classmethod
    def int6(cls, group_size: int = 128, rounding: str = "nearest-even", **kw) -> "FlashConfig":
        s1, s2 = int6_flash_pair(group_size=group_size, rounding=rounding)
        return cls(stage1_codec=s1, stage2_codec=s2, **kw)

    @classmethod
    def from_bits(cls, bits: int, group_size: int = 128, **kw) -> "FlashConfig":  # collectives.py:100-109
        if bits == 16:
            return cls.uniform(PASSTHROUGH_FP16, **kw)
        if bits == 6:
            return cls.int6(group_size=group_size, **kw)
        if bits in (4, 8):
            return cls.uniform(CodecConfig(bits=bits, group_size=group_size), **kw)
        raise ConfigError(f"no preset for {bits} effective bits")


@dataclass
class CollectiveRun:
    """Outputs plus the counters of collectives.py:112-127."""

    method: str
    outputs: list
    ledger: TrafficLedger
    reduce_steps: int
    gather_steps: int
    qdq_passes: int
    reduce_elems_per_rank: int
    gather_elems_per_rank: int

    @property
    def wire_bytes_per_rank(self) -> int:
        return self.ledger.rank_bytes_sent(0)


def sequential_sum(parts: Sequence[torch.Tensor]) -> torch.Tensor:
    """fp32, ascending rank order (collectives.py:182-187)."""
    acc = parts[0].to(torch.float32).clone()
    for p in parts[1:]:
        acc += p.to(device=acc.device, dtype=torch.float32)
    return acc


def _rank_tensors(tensors: Sequence) -> tuple[list, tuple, int]:
    if len(tensors) == 0:
        raise ProtocolError("need at least one rank tensor")
    shape = tuple(tensors[0].shape) if hasattr(tensors[0], "shape") else (len(tensors[0]),)
    flats = [as_device_tensor(t) for t in tensors]
    m = flats[0].numel()
    for r, f in enumerate(flats):
        if f.numel() != m:
            raise ProtocolError(f"rank {r} tensor length {f.numel()} != rank 0 length {m}")
        if f.dtype != flats[0].dtype:
            raise ProtocolError(f"rank {r} dtype {f.dtype} != rank 0 dtype {flats[0].dtype}")
    if m == 0:
        raise DomainError("rank tensors must be nonempty")
    return flats, shape, m


def _check_topology(topology, n: int) -> None:
    if topology is not None and topology.world_size != n:
        raise ConfigError(f"topology world_size {topology.world_size} != {n} rank tensors")


_COMMS: dict = {}


def local_comm(devices: Sequence[int], slot_bytes: int) -> FlashComm:
    """Cached one-process communicator for `devices` with >= slot_bytes slots."""
    key = tuple(devices)
    comm = _COMMS.get(key)
    if comm is None or comm.slot_bytes < slot_bytes:
        if comm is not None:
            comm.close()
        comm = FlashComm.local(list(devices), slot_bytes)
        _COMMS[key] = comm
    return comm


def flash_all_reduce(tensors: Sequence, cfg: FlashConfig, topology: Optional[FabricTopology] = None,
                     timeout: float = DEFAULT_TIMEOUT_S, *, out_dtype: Optional[torch.dtype] = None,
                     comm: Optional[FlashComm] = None, outs: Optional[Sequence] = None) -> CollectiveRun:
    """Two-step quantized all-reduce (collectives.py:321-402) on the GPU.

    Outputs are new tensors of the input shape and, unless `out_dtype` is
    given, the input dtype (float32 output equals the reference bit for bit;
    bf16/fp16 output is its round-to-nearest-even). Blocks until done and
    raises like the reference: DomainError for NaN/inf input, ProtocolError
    when a rank never arrives within `timeout` seconds.

    Host tensors / arrays in (the reference's own call shape) give host
    tensors out: one blocking call pipelines the H2D copy, the all-reduce and
    the D2H copy chunk by chunk (fc_flash_all_reduce_host); `outs` may supply
    the host output tensors (flat, n elements each) to reuse pinned buffers.
    """
    if cfg.rotation is None and _all_host(tensors):
        return _flash_all_reduce_host(tensors, cfg, topology, timeout, out_dtype, comm, outs)
    if outs is not None:
        raise ConfigError("outs= is for host tensors (device callers use FlashComm.all_reduce_local)")
    flats, shape, m = _rank_tensors(tensors)
    n = len(flats)
    _check_topology(topology, n)
    odt = out_dtype or flats[0].dtype
    if n == 1:  # collectives.py:340-341
        return CollectiveRun("flash", [flats[0].to(odt).clone().reshape(shape)], TrafficLedger.zeros(1), 0, 0, 0, 0, 0)
    chunk = cfg.resolve_chunk_size(n)  # ConfigError exactly like the reference
    seg = -(-m // n)
    devices = [f.device.index for f in flats]
    if comm is None:
        comm = local_comm(devices, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_timeout(timeout if timeout is not None else 3600.0)
    if cfg.rotation is not None and comm.rotation_fusable(m, cfg, cfg.rotation):
        # the rotation fused into the lane-8 kernels: H(D x) in the scatter / reduce prologue,
        # D(H y) in the reduce / gather epilogue (fc_l8.cuh), no float32 copies of the tensors
        rot = cfg.rotation
        signs = [rot._device_signs(f.device) for f in flats]  # alive until the call has synchronised
        comm.set_rotation(rot, signs)
        try:
            outs = comm.all_reduce_local(flats, cfg, out_dtype=odt, check=True)
        finally:
            comm.set_rotation(None)
    elif cfg.rotation is not None:
        # not fusable here (rotation block > 256, segment not a multiple of it, or a group size
        # the lane-8 kernels do not take): rotate the zero-padded rank tensors (float32),
        # all-reduce, rotate back, trim -- three passes
        from .rotation import hadamard_apply, hadamard_inverse

        rot = cfg.rotation
        rins = [hadamard_apply(f, rot, n * seg) for f in flats]
        routs = comm.all_reduce_local(rins, cfg, out_dtype=torch.float32, check=True)
        outs = [hadamard_inverse(o, rot, out_dtype=odt, n_out=m) for o in routs]
        torch.cuda.synchronize(flats[0].device)
    else:
        outs = comm.all_reduce_local(flats, cfg, out_dtype=odt, check=True)
    qdq = int(not cfg.stage1_codec.is_passthrough) + int(not cfg.stage2_codec.is_passthrough)
    return CollectiveRun(
        method="flash",
        outputs=[o.reshape(shape) for o in outs],
        ledger=flash_ledger(n, seg, chunk // n, cfg.stage1_codec, cfg.stage2_codec),
        reduce_steps=1,
        gather_steps=1,
        qdq_passes=qdq,
        reduce_elems_per_rank=(n - 1) * seg,
        gather_elems_per_rank=(n - 1) * seg,
    )


def _all_host(tensors: Sequence) -> bool:
    return len(tensors) > 0 and all(not (isinstance(t, torch.Tensor) and t.is_cuda) for t in tensors)


def _flash_all_reduce_host(tensors, cfg, topology, timeout, out_dtype, comm, outs=None) -> CollectiveRun:
    """Host arrays in, new host arrays out (the reference's own call shape):
    one blocking C-ABI call (fc_flash_all_reduce_host) pipelines the chunked
    H2D copy, the flash all-reduce and the D2H copy on the communicator's
    streams; the result equals the device-buffer call bit for bit."""
    flats, shape, m = _host_rank_tensors(tensors)
    n = len(flats)
    _check_topology(topology, n)
    odt = out_dtype or flats[0].dtype
    if n == 1:  # collectives.py:340-341
        return CollectiveRun("flash", [flats[0].to(odt).clone().reshape(shape)], TrafficLedger.zeros(1), 0, 0, 0, 0, 0)
    chunk = cfg.resolve_chunk_size(n)  # ConfigError exactly like the reference
    seg = -(-m // n)
    dev = torch.cuda.current_device()
    if comm is None:
        comm = local_comm([dev] * n, slot_bytes_for(seg, cfg.stage1_codec, cfg.stage2_codec))
    comm.set_timeout(timeout if timeout is not None else 3600.0)
    outs = comm.all_reduce_host(flats, cfg, out_dtype=odt, outs=outs)
    qdq = int(not cfg.stage1_codec.is_passthrough) + int(not cfg.stage2_codec.is_passthrough)
    return CollectiveRun(
        method="flash",
        outputs=[o.reshape(shape) if o is not None else None for o in outs],
        ledger=flash_ledger(n, seg, chunk // n, cfg.stage1_codec, cfg.stage2_codec),
        reduce_steps=1,
        gather_steps=1,
        qdq_passes=qdq,
        reduce_elems_per_rank=(n - 1) * seg,
        gather_elems_per_rank=(n - 1) * seg,
    )


def _host_rank_tensors(tensors: Sequence) -> tuple[list, tuple, int]:
    if len(tensors) == 0:
        raise ProtocolError("need at least one rank tensor")
    shape = tuple(tensors[0].shape) if hasattr(tensors[0], "shape") else (len(tensors[0]),)
    flats = [as_host_tensor(t) for t in tensors]
    m = flats[0].numel()
    for r, f in enumerate(flats):
        if f.numel() != m:
            raise ProtocolError(f"rank {r} tensor length {f.numel()} != rank 0 length {m}")
        if f.dtype != flats[0].dtype:
            raise ProtocolError(f"rank {r} dtype {f.dtype} != rank 0 dtype {flats[0].dtype}")
    if m == 0:
        raise DomainError("rank tensors must be nonempty")
    return flats, shape, m


def all_reduce_exact(tensors: Sequence, topology: Optional[FabricTopology] = None,
                     timeout: float = DEFAULT_TIMEOUT_S) -> CollectiveRun:
    """The accuracy yardstick (collectives.py:190-241): raw fp32, rank-ordered
    sum. Not a hot path; plain device arithmetic."""
    flats, shape, m = _rank_tensors(tensors)
    n = len(flats)
    _check_topology(topology, n)
    if n == 1:
        return CollectiveRun("exact", [flats[0].float().clone().reshape(shape)], TrafficLedger.zeros(1), 0, 0, 0, 0, 0)
    red = sequential_sum(flats)
    seg = -(-m // n)
    led = TrafficLedger.zeros(n)
    for s in range(n):
        for r in range(n):
            if s != r:
                led.bytes_sent[s][r] = 2 * seg * 4
                led.messages[s][r] = 2
    led.steps = 2
    outs = [red.to(f.device).reshape(shape) for f in flats]
    return CollectiveRun("exact", outs, led, 1, 1, 0, (n - 1) * seg, (n - 1) * seg)


def run_collective(method: str, tensors: Sequence, *, codec: Optional[CodecConfig] = None,
                   flash: Optional[FlashConfig] = None, topology: Optional[FabricTopology] = None,
                   timeout: float = DEFAULT_TIMEOUT_S) -> CollectiveRun:
    """Dispatch by method name (collectives.py:445-465)."""
    if method == "exact":
        return all_reduce_exact(tensors, topology=topology, timeout=timeout)
    if method == "flash":
        if flash is None:
            raise ConfigError("flash method needs a FlashConfig")
        return flash_all_reduce(tensors, flash, topology=topology, timeout=timeout)
    if method == "ring":
        raise ConfigError("the ring method is the uncompressed baseline on B200: use "
                          "torch.distributed.all_reduce (NCCL)")
    raise ConfigError(f"unknown method {method!r}, expected one of {METHODS}")
