"""Communicator: the B200 replacement of the reference's simulated fabric
(/root/reference/pkg/src/qcollectives/fabric.py:111-246).

A `FlashComm` owns, per rank, one device block holding N stage-1 receive
slots, N stage-2 gather slots, per-tile arrival flags and an error word
(layout: include/flashcomm.h, csrc/fc_flash.cuh). Peers write into it
directly over NVLink: P2P between the GPUs of one process (`local`), or CUDA
IPC between one process per GPU (`from_process_group`; handles are exchanged
over torch.distributed). What the reference fabric guaranteed is kept: a
rank that never arrives surfaces as ProtocolError naming the stuck pair
(fabric.py:158-178, timeout default 5 s), and per-link wire bytes follow the
reference ledger formula (collectives.py:152-157, costmodel.py:122-128).
"""

from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

from . import _lib
from .codec import CodecConfig, QuantizedTensor, fc_dtype
from .errors import ConfigError, DomainError, ProtocolError

DEFAULT_TIMEOUT_S = 5.0  # fabric.py:132


@dataclass(frozen=True)
class FabricTopology:
    """Signature-compatible stand-in for fabric.py:33-48 (flat homogeneous
    topology). On B200 the link model is NVLink 5 through NVSwitch; the
    measured topology is `FlashComm.topology()`."""

    world_size: int
    link_bandwidth: float = 900e9
    base_latency: float = 2e-6
    qdq_cost: float = 0.0

    def __post_init__(self) -> None:
        if int(self.world_size) < 1:
            raise ConfigError(f"world_size must be >= 1, got {self.world_size}")
        if not self.link_bandwidth > 0:
            raise ConfigError("link_bandwidth must be positive")
        if self.base_latency < 0 or self.qdq_cost < 0:
            raise ConfigError("latencies must be nonnegative")


@dataclass
class TrafficLedger:
    """Per-link byte/message counters (fabric.py:51-91). Filled analytically
    from the call's piece layout; GPU kernels move exactly these bytes."""

    bytes_sent: list
    messages: list
    steps: int = 0

    @classmethod
    def zeros(cls, n: int) -> "TrafficLedger":
        return cls([[0] * n for _ in range(n)], [[0] * n for _ in range(n)])

    @property
    def world_size(self) -> int:
        return len(self.bytes_sent)

    def rank_bytes_sent(self, rank: int) -> int:
        return sum(self.bytes_sent[rank])

    def total_bytes(self) -> int:
        return sum(map(sum, self.bytes_sent))

    def to_json_dict(self) -> dict:
        return {"bytes_sent": self.bytes_sent, "messages": self.messages, "steps": self.steps}


def piece_layout(seg: int, piece: int):
    """(offset, length) pieces of one rank segment (collectives.py:152-157)."""
    off = 0
    while off < seg:
        yield off, min(piece, seg - off)
        off += piece


def flash_ledger(n_ranks: int, seg: int, piece: int, stage1: CodecConfig, stage2: CodecConfig) -> TrafficLedger:
    """Bytes/messages each directed pair carries in flash_all_reduce: per piece
    one stage-1 and one stage-2 message (collectives.py:359-385)."""
    per_pair = 0
    msgs = 0
    for _, plen in piece_layout(seg, piece):
        per_pair += stage1.wire_byte_len(plen) + stage2.wire_byte_len(plen)
        msgs += 2
    led = TrafficLedger.zeros(n_ranks)
    for s in range(n_ranks):
        for r in range(n_ranks):
            if s != r:
                led.bytes_sent[s][r] = per_pair
                led.messages[s][r] = msgs
    led.steps = 2
    return led


TILE_ELEMS = 8192  # elements per CTA tile (csrc/fc_common.cuh kTileElems)


def slot_bytes_for(seg: int, *codecs: CodecConfig) -> int:
    """Smallest slot capacity holding one round of a whole segment (rounds
    are cut at multiples of the tile and of every group size)."""
    unit = TILE_ELEMS
    for c in codecs:
        if not c.is_passthrough:
            unit = math.lcm(unit, c.group_size)
    n = -(-seg // unit) * unit
    need = 4096
    for c in codecs:
        need = max(need, int(c.device_layout(n).total_bytes))
    return int(math.ceil(need / 4096.0) * 4096)


def exchange_handles(my_handle: bytes, group=None) -> bytes:
    """All-gather every rank's IPC handle in rank order over torch.distributed
    (any backend: gloo for CPU tests, nccl on the box)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    got: list = [None] * world
    dist.all_gather_object(got, bytes(my_handle), group=group)
    for r, h in enumerate(got):
        if not isinstance(h, (bytes, bytearray)) or len(h) != len(my_handle):
            raise ProtocolError(f"rank {r} sent a malformed IPC handle")
    return b"".join(bytes(h) for h in got)


def _check_out(o: torch.Tensor, n: int, dtype: torch.dtype, device: int, what: str) -> None:
    """Caller-supplied output buffers: the kernels write n elements of `dtype`
    through a raw pointer, so size, dtype, layout and device are checked here."""
    if not isinstance(o, torch.Tensor):
        raise DomainError(f"{what} must be a tensor")
    if o.numel() != n:
        raise DomainError(f"{what} holds {o.numel()} elements, expected {n}")
    if o.dtype != dtype:
        raise DomainError(f"{what} dtype {o.dtype} != {dtype}")
    if not o.is_contiguous():
        raise DomainError(f"{what} must be contiguous")
    if o.get_device() != device:
        raise DomainError(f"{what} must live on cuda:{device}")


def _device_index(d) -> int:
    if isinstance(d, torch.device):
        return d.index if d.index is not None else torch.cuda.current_device()
    if isinstance(d, str):
        return _device_index(torch.device(d))
    return int(d)


@functools.lru_cache(maxsize=None)
def _ptr_array(n: int):
    return C.c_void_p * n


@functools.lru_cache(maxsize=256)
def _cfg_struct(cfg) -> _lib.fc_flash_cfg:
    return _lib.fc_flash_cfg(cfg.stage1_codec.to_fc(), cfg.stage2_codec.to_fc(),
                             int(cfg.chunk_size) if cfg.chunk_size is not None else 0)


class FlashComm:
    """Peer-buffer manager + topology + flag protocol (see module doc)."""

    def __init__(self, handle: C.c_void_p, world: int, devices: list, rank: Optional[int], slot_bytes: int):
        self._h = handle
        self.world_size = world
        self.devices = devices
        self.rank = rank  # None for a local (one-process) communicator
        self.slot_bytes = slot_bytes

    # ---------------------------------------------------------------- creation
    @classmethod
    def local(cls, devices: Sequence, slot_bytes: int) -> "FlashComm":
        devs = [_device_index(d) for d in devices]
        n = len(devs)
        if not 1 <= n <= _lib.FC_MAX_RANKS:
            raise ConfigError(f"world_size must be in 1..{_lib.FC_MAX_RANKS}, got {n}")
        arr = (C.c_int32 * n)(*devs)
        h = C.c_void_p()
        _lib.check(_lib.lib().fc_comm_create_local(n, arr, int(slot_bytes), C.byref(h)))
        return cls(h, n, devs, None, int(slot_bytes))

    @classmethod
    def from_process_group(cls, group=None, device=None, slot_bytes: int = 64 << 20) -> "FlashComm":
        """One process per GPU (torchrun): allocate, exchange IPC handles, map peers."""
        import torch.distributed as dist

        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        dev = _device_index(device if device is not None else torch.cuda.current_device())
        h = C.c_void_p()
        _lib.check(_lib.lib().fc_comm_create_ipc(world, rank, dev, int(slot_bytes), C.byref(h)))
        comm = cls(h, world, [dev] * world, rank, int(slot_bytes))
        try:
            mine = (C.c_uint8 * _lib.FC_IPC_HANDLE_BYTES)()
            _lib.check(_lib.lib().fc_comm_ipc_handle(h, mine))
            allh = exchange_handles(bytes(mine), group)
            buf = (C.c_uint8 * len(allh)).from_buffer_copy(allh)
            _lib.check(_lib.lib().fc_comm_ipc_open(h, buf))
            dist.barrier(group)
        except Exception:
            comm.close()
            raise
        return comm

    def close(self) -> None:
        if self._h:
            _lib.lib().fc_comm_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- options
    def set_option(self, option: int, value: int) -> None:
        _lib.check(_lib.lib().fc_comm_set_option(self._h, int(option), int(value)))

    def get_option(self, option: int) -> int:
        v = C.c_int64()
        _lib.check(_lib.lib().fc_comm_get_option(self._h, int(option), C.byref(v)))
        return v.value

    def set_timeout(self, seconds: float) -> None:
        self.set_option(_lib.OPT_TIMEOUT_MS, max(1, int(round(seconds * 1000))))

    # ---------------------------------------------------------------- fused rotation
    def rotation_fusable(self, n: int, cfg, block) -> bool:
        """Whether a run of n elements per rank can fuse `block` (rotation.HadamardBlock)
        into its prologue / epilogue (fc_flash_rotation_fusable)."""
        cs = self._cfg(cfg)
        return bool(_lib.lib().fc_flash_rotation_fusable(self._h, int(n), C.byref(cs), int(block.dimension)))

    def set_rotation(self, block, signs: Optional[Sequence[Optional[torch.Tensor]]] = None) -> None:
        """Fuse `block` into the next runs (None clears). signs: per-rank device tensors of the
        seeded +-1 diagonal on the ranks' devices (block.signs()), or None."""
        L = _lib.lib()
        if block is None:
            _lib.check(L.fc_comm_set_rotation(self._h, -1, 0, 1, None))
            return
        for r in range(self.world_size):
            if self.rank is not None and r != self.rank:
                continue
            sp = signs[r].data_ptr() if signs is not None and signs[r] is not None else None
            _lib.check(L.fc_comm_set_rotation(self._h, r, int(block.dimension), int(bool(block.normalize)), sp))

    # ---------------------------------------------------------------- calls
    @staticmethod
    def _cfg(cfg) -> _lib.fc_flash_cfg:
        # FlashConfig is frozen (hashable): the C struct is built once per config
        # (the C side takes it as const), keeping the per-call host path short
        return _cfg_struct(cfg)

    def all_reduce_local(self, ins: Sequence[torch.Tensor], cfg, outs: Optional[Sequence[torch.Tensor]] = None,
                         out_dtype: Optional[torch.dtype] = None, check: bool = True) -> list:
        """One process, all ranks: ins[r] lives on devices[r] (flat, contiguous)."""
        if self.rank is not None:
            raise ConfigError("all_reduce_local needs a local communicator")
        if len(ins) != self.world_size:
            raise ProtocolError(f"expected {self.world_size} rank tensors, got {len(ins)}")
        n = ins[0].numel()
        dt = ins[0].dtype
        for r, t in enumerate(ins):
            if t.numel() != n:
                raise ProtocolError(f"rank {r} tensor length {t.numel()} != rank 0 length {n}")
            if t.dtype != dt:
                raise ProtocolError(f"rank {r} dtype {t.dtype} != rank 0 dtype {dt}")
            if t.get_device() != self.devices[r]:  # -1 for host tensors
                raise DomainError(f"rank {r} tensor must live on cuda:{self.devices[r]}")
            if not t.is_contiguous():
                raise DomainError(f"rank {r} tensor must be contiguous")
        odt = out_dtype or dt
        fc_dtype(odt)
        if outs is None:
            outs = [torch.empty(n, dtype=odt, device=t.device) for t in ins]
        else:
            if len(outs) != self.world_size:
                raise ProtocolError(f"expected {self.world_size} output tensors, got {len(outs)}")
            for r, o in enumerate(outs):
                _check_out(o, n, odt, self.devices[r], f"rank {r} output")
        N = self.world_size
        arr = _ptr_array(N)
        pin = arr(*[t.data_ptr() for t in ins])
        pout = arr(*[o.data_ptr() for o in outs])
        streams = {}  # one current-stream lookup per distinct device
        for d in self.devices:
            if d not in streams:
                streams[d] = torch.cuda.current_stream(d).cuda_stream
        pst = arr(*[streams[d] for d in self.devices])
        c = self._cfg(cfg)
        _lib.check(_lib.lib().fc_flash_all_reduce_local(self._h, pin, pout, n, fc_dtype(dt), fc_dtype(odt),
                                                        C.byref(c), pst))
        if check:
            self.check()
        return list(outs)

    def all_reduce_host(self, ins: Sequence[torch.Tensor], cfg, out_dtype: Optional[torch.dtype] = None,
                        read_back: Optional[Sequence[bool]] = None,
                        outs: Optional[Sequence[Optional[torch.Tensor]]] = None) -> list:
        """Blocking all-reduce of one HOST tensor per rank (the reference's
        arrays-in / new-arrays-out call): chunked H2D, the flash all-reduce per
        chunk and chunked D2H overlap on the communicator's own streams
        (fc_flash_all_reduce_host). Returns new pinned host tensors (None for
        ranks with read_back[r] False), or fills `outs` (host tensors of n
        elements, None to skip a rank). Pinned buffers copy at full PCIe rate."""
        if self.rank is not None:
            raise ConfigError("all_reduce_host needs a local communicator")
        if len(ins) != self.world_size:
            raise ProtocolError(f"expected {self.world_size} rank tensors, got {len(ins)}")
        n = ins[0].numel()
        dt = ins[0].dtype
        for r, t in enumerate(ins):
            if t.numel() != n:
                raise ProtocolError(f"rank {r} tensor length {t.numel()} != rank 0 length {n}")
            if t.dtype != dt:
                raise ProtocolError(f"rank {r} dtype {t.dtype} != rank 0 dtype {dt}")
            if t.is_cuda:
                raise DomainError(f"rank {r} tensor must be a host tensor")
            if not t.is_contiguous():
                raise DomainError(f"rank {r} tensor must be contiguous")
        odt = out_dtype or dt
        N = self.world_size
        if outs is None:
            outs = [torch.empty(n, dtype=odt, pin_memory=True) if (read_back is None or read_back[r]) else None
                    for r in range(N)]
        else:
            if len(outs) != N:
                raise ProtocolError(f"expected {N} output tensors, got {len(outs)}")
            for r, o in enumerate(outs):
                if o is None:
                    continue
                if o.is_cuda or not o.is_contiguous() or o.numel() != n or o.dtype != odt:
                    raise DomainError(f"rank {r} output must be a contiguous host {odt} tensor of {n} elements")
            outs = list(outs)
        arr = _ptr_array(N)
        pin = arr(*[t.data_ptr() for t in ins])
        pout = arr(*[o.data_ptr() if o is not None else None for o in outs])
        _lib.check(_lib.lib().fc_flash_all_reduce_host(self._h, pin, pout, n, fc_dtype(dt), fc_dtype(odt),
                                                       C.byref(self._cfg(cfg))))
        return outs

    def all_reduce_host_rank(self, tensor: torch.Tensor, cfg, out: Optional[torch.Tensor] = None,
                             out_dtype: Optional[torch.dtype] = None, read_back: bool = True):
        """Per-rank host-buffer form (IPC world): this rank's host tensor in,
        a new (or the given `out`) host tensor out, chunked H2D / all-reduce /
        D2H overlapped (fc_flash_all_reduce_host_rank). Blocking; every rank
        calls it with the same numel / cfg / FC_OPT_HOST_CHUNK_BYTES."""
        if self.rank is None:
            raise ConfigError("all_reduce_host_rank needs an IPC communicator (from_process_group)")
        if tensor.is_cuda or not tensor.is_contiguous():
            raise DomainError("tensor must be a contiguous host tensor")
        n = tensor.numel()
        odt = out_dtype or tensor.dtype
        if out is None and read_back:
            out = torch.empty(n, dtype=odt, pin_memory=True)
        if out is not None and (out.is_cuda or not out.is_contiguous() or out.numel() != n or out.dtype != odt):
            raise DomainError(f"out must be a contiguous host {odt} tensor of {n} elements")
        _lib.check(_lib.lib().fc_flash_all_reduce_host_rank(
            self._h, tensor.data_ptr(), out.data_ptr() if out is not None else None, n, fc_dtype(tensor.dtype),
            fc_dtype(odt), C.byref(self._cfg(cfg))))
        return out

    def all_reduce(self, tensor: torch.Tensor, cfg, out: Optional[torch.Tensor] = None,
                   out_dtype: Optional[torch.dtype] = None, check: bool = False) -> torch.Tensor:
        """Per-rank form (IPC world): every rank calls with equal numel/cfg.
        out may be `tensor` (in place). Asynchronous unless check=True."""
        if self.rank is None:
            raise ConfigError("all_reduce needs an IPC communicator (from_process_group)")
        if tensor.get_device() != self.devices[self.rank]:
            raise DomainError(f"tensor must live on cuda:{self.devices[self.rank]}")
        if not tensor.is_contiguous():
            raise DomainError("tensor must be contiguous")
        odt = out_dtype or tensor.dtype
        fc_dtype(odt)
        if out is None:
            out = torch.empty_like(tensor, dtype=odt)
        else:
            _check_out(out, tensor.numel(), odt, self.devices[self.rank], "out")
        c = self._cfg(cfg)
        st = torch.cuda.current_stream(tensor.device).cuda_stream
        _lib.check(_lib.lib().fc_flash_all_reduce(self._h, tensor.data_ptr(), out.data_ptr(), tensor.numel(),
                                                  fc_dtype(tensor.dtype), fc_dtype(odt), C.byref(c), st))
        if check:
            self.check()
        return out

    def teardown_check(self) -> None:
        """fabric.py:228-236: ProtocolError when the ranks did not all complete the same
        number of rounds (messages left unconsumed). IPC communicators; call after the
        ranks' last collective."""
        _lib.check(_lib.lib().fc_comm_teardown_check(self._h))

    def check(self, rank: int = -1) -> None:
        """Synchronize and raise the device-side error of `rank` (all if -1)."""
        _lib.check(_lib.lib().fc_comm_check(self._h, int(rank)))

    # ---------------------------------------------------------------- debug / parity
    def slot(self, rank: int, stage: int, src: int, config: CodecConfig) -> QuantizedTensor:
        """Stage-1 receive slot [src] or stage-2 gather slot [src] of `rank`
        as a QuantizedTensor (the last round of the last call)."""
        L = _lib.fc_layout()
        _lib.check(_lib.lib().fc_comm_slot(self._h, rank, stage, src, None, C.byref(L)))
        dev = torch.device("cuda", self.devices[rank] if self.rank is None else self.devices[self.rank])
        raw = torch.empty(int(L.total_bytes), dtype=torch.uint8, device=dev)
        _lib.check(_lib.lib().fc_comm_slot(self._h, rank, stage, src, raw.data_ptr(), C.byref(L)))
        qt = QuantizedTensor.__new__(QuantizedTensor)
        qt.config = config
        qt.element_count = int(L.elements)
        qt._buf = raw
        qt._layout = L
        qt.codes = raw[: L.codes_bytes]
        qt.scales_f16 = (raw[L.scales_offset: L.scales_offset + 2 * L.groups].view(torch.float16)
                         if not config.is_passthrough else torch.empty(0, dtype=torch.float16, device=dev))
        qt.zeros = raw[L.zeros_offset: L.zeros_offset + L.groups] if (config.is_int and not config.symmetric) else None
        return qt

    def topology(self) -> dict:
        N = self.world_size
        acc = (C.c_int32 * (N * N))()
        mc = C.c_int32()
        _lib.check(_lib.lib().fc_comm_topology(self._h, acc, C.byref(mc)))
        names = sorted({torch.cuda.get_device_name(d) for d in set(self.devices)})
        return {"world_size": N, "devices": list(self.devices), "device_names": names,
                "peer_access": [[int(acc[a * N + b]) for b in range(N)] for a in range(N)],
                "multicast_supported": bool(mc.value), "ipc": self.rank is not None,
                "nvlink": nvlink_topology(sorted(set(self.devices)))}


def nvlink_topology(devices: Sequence[int]) -> dict:
    """NVML view of the box (one 8xB200 NVSwitch node): per CUDA device its PCI bus id,
    active NVLink links and their remote PCI ids (NVSwitch ports on an HGX B200), and the
    NVML P2P status between the devices. Missing NVML or NVLink reports empty fields
    (a single-GPU box has no active links); it never raises."""
    out = {"nvml": False, "devices": {}}
    try:
        import pynvml as nv

        nv.nvmlInit()
    except Exception as e:  # pragma: no cover - NVML absent
        out["error"] = repr(e)
        return out
    out["nvml"] = True
    try:
        handles = {}
        for d in devices:
            props = torch.cuda.get_device_properties(d)
            h = nv.nvmlDeviceGetHandleByUUID(f"GPU-{props.uuid}")  # CUDA ordinal -> NVML handle
            handles[d] = h
            pci = nv.nvmlDeviceGetPciInfo(h)
            bus = pci.busId.decode() if isinstance(pci.busId, bytes) else str(pci.busId)
            links = []
            for ln in range(18):  # NVML_NVLINK_MAX_LINKS on Blackwell
                try:
                    if nv.nvmlDeviceGetNvLinkState(h, ln) == nv.NVML_FEATURE_ENABLED:
                        rp = nv.nvmlDeviceGetNvLinkRemotePciInfo_v2(h, ln)
                        links.append({"link": ln, "remote_bus": rp.busId.decode() if isinstance(rp.busId, bytes)
                                      else str(rp.busId)})
                except Exception:
                    break
            out["devices"][str(d)] = {"pci_bus_id": bus, "nvlink_active": len(links), "links": links}
        p2p = {}
        for a in devices:
            for b in devices:
                if a < b:
                    try:
                        st = nv.nvmlDeviceGetP2PStatus(handles[a], handles[b], nv.NVML_P2P_CAPS_INDEX_NVLINK)
                        p2p[f"{a}-{b}"] = "ok" if st == nv.NVML_P2P_STATUS_OK else f"status {st}"
                    except Exception as e:
                        p2p[f"{a}-{b}"] = repr(e)
        out["p2p_nvlink"] = p2p
    except Exception as e:
        out["error"] = repr(e)
    finally:
        try:
            nv.nvmlShutdown()
        except Exception:
            pass
    return out
