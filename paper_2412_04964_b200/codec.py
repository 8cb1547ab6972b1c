"""Group codec on the GPU: the reference's `qcollectives.codec` interface
(/root/reference/pkg/src/qcollectives/codec.py) over CUDA tensors.

Names, fields, validation and error behaviour follow the reference:
`CodecConfig` (codec.py:45-159), `PASSTHROUGH_FP16` (:162),
`QuantizedTensor` (:165-219), `quantize` (:292-329), `dequantize`
(:354-384), `mse` (:387-393), `codec_from_name` (:396-420),
`int6_flash_pair` (:423-429). Arithmetic runs in libflashcomm's sm_100a
kernels and is bit-exact with the reference (codes, fp16 scales, zeros and
dequantized values).
"""

from __future__ import annotations

import ctypes as C
import re
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, DomainError, IntegrityError

ROUNDING_MODES = ("nearest-even", "ceil")
FLOAT_FORMATS = ("e4m3", "e5m2", "e2m1", "fp16")
_MINIFLOAT_BITS = {"e4m3": 8, "e5m2": 8, "e2m1": 4}

_TORCH_DTYPES = {
    torch.float32: _lib.DTYPE_F32,
    torch.float16: _lib.DTYPE_F16,
    torch.bfloat16: _lib.DTYPE_BF16,
}


def fc_dtype(dt: torch.dtype) -> int:
    try:
        return _TORCH_DTYPES[dt]
    except KeyError:
        raise DomainError(f"unsupported dtype {dt}; expected float32, float16 or bfloat16") from None


@dataclass(frozen=True)
class CodecConfig:
    """One quantization scheme (codec.py:45-73): exactly one of `bits`
    (2..8 integer codes) or `number_format` (e4m3 / e5m2 / e2m1 group-scaled
    minifloats, codec.py:332-351, or the fp16 passthrough)."""

    bits: Optional[int] = None
    number_format: Optional[str] = None
    group_size: int = 128
    symmetric: bool = False
    rounding: str = "nearest-even"
    scale_floor: float = 1e-8

    def __post_init__(self) -> None:
        if (self.bits is None) == (self.number_format is None):
            raise ConfigError("set exactly one of bits or number_format")
        if self.bits is not None and not 2 <= int(self.bits) <= 8:
            raise ConfigError(f"bits must be in 2..8, got {self.bits}")
        if self.number_format is not None and self.number_format not in FLOAT_FORMATS:
            raise ConfigError(f"number_format must be one of {FLOAT_FORMATS}")
        if int(self.group_size) < 1:
            raise ConfigError("group_size must be >= 1")
        if self.rounding not in ROUNDING_MODES:
            raise ConfigError(f"rounding must be one of {ROUNDING_MODES}")
        if not self.scale_floor > 0:
            raise ConfigError("scale_floor must be positive")

    is_passthrough = property(lambda self: self.number_format == "fp16")
    is_minifloat = property(lambda self: self.number_format in _MINIFLOAT_BITS)
    is_int = property(lambda self: self.bits is not None)

    @property
    def code_bits(self) -> int:
        if self.is_passthrough:
            return 16
        if self.is_minifloat:
            return _MINIFLOAT_BITS[self.number_format]
        return int(self.bits)

    @property
    def storage_bits(self) -> int:  # codec.py:98-103
        if self.is_passthrough:
            return 16
        return 4 if self.code_bits <= 4 else 8

    @property
    def metadata_bytes_per_group(self) -> int:  # codec.py:105-112
        if self.is_passthrough:
            return 0
        return 3 if (self.is_int and not self.symmetric) else 2

    @property
    def label(self) -> str:
        if self.number_format is not None:
            return self.number_format
        return f"int{self.bits}{'sym' if self.symmetric else 'asym'}"

    def group_count(self, element_count: int) -> int:
        return 0 if self.is_passthrough else -(-element_count // self.group_size)

    def wire_byte_len(self, element_count: int) -> int:  # codec.py:128-133
        if self.is_passthrough:
            return 2 * element_count
        packed = (element_count * self.storage_bits + 7) // 8
        return packed + self.group_count(element_count) * self.metadata_bytes_per_group

    def to_json_dict(self) -> dict:
        d: dict = {"group_size": self.group_size, "symmetric": self.symmetric,
                   "rounding": self.rounding, "scale_floor": self.scale_floor}
        if self.bits is not None:
            d["bits"] = self.bits
        else:
            d["format"] = self.number_format
        return d

    @classmethod
    def from_json_dict(cls, d: dict) -> "CodecConfig":
        extra = set(d) - {"bits", "format", "group_size", "symmetric", "rounding", "scale_floor"}
        if extra:
            raise ConfigError(f"unknown codec keys: {sorted(extra)}")
        return cls(bits=d.get("bits"), number_format=d.get("format"),
                   group_size=d.get("group_size", 128), symmetric=d.get("symmetric", False),
                   rounding=d.get("rounding", "nearest-even"), scale_floor=d.get("scale_floor", 1e-8))

    # ---- C ABI view
    def to_fc(self) -> _lib.fc_codec:
        if self.is_minifloat:
            return _lib.fc_codec(_lib.KIND_MINIFLOAT, self.code_bits, int(self.group_size), 0, 0,
                                 _lib.MINIFLOAT_FORMAT_IDS[self.number_format], float(self.scale_floor))
        if self.is_passthrough:
            return _lib.fc_codec(_lib.KIND_FP16, 16, 1, 0, 0, 0, self.scale_floor)
        return _lib.fc_codec(_lib.KIND_INT, int(self.bits), int(self.group_size), int(bool(self.symmetric)),
                             _lib.ROUND_CEIL if self.rounding == "ceil" else _lib.ROUND_NEAREST_EVEN, 0,
                             float(self.scale_floor))

    def device_layout(self, element_count: int) -> _lib.fc_layout:
        out = _lib.fc_layout()
        c = self.to_fc()
        _lib.check(_lib.lib().fc_codec_layout(C.byref(c), int(element_count), C.byref(out)))
        return out


PASSTHROUGH_FP16 = CodecConfig(number_format="fp16")


def codec_from_name(name: str, group_size: int = 128, rounding: str = "nearest-even",
                    scale_floor: float = 1e-8) -> CodecConfig:
    """intN[asym|sym] / e4m3 / e5m2 / e2m1 / fp16 (codec.py:396-420)."""
    key = name.strip().lower()
    if key in ("fp16", "passthrough"):
        return PASSTHROUGH_FP16
    if key in FLOAT_FORMATS:
        return CodecConfig(number_format=key, group_size=group_size, rounding=rounding, scale_floor=scale_floor)
    m = re.fullmatch(r"int(\d+)(asym|sym)?", key)
    if m:
        return CodecConfig(bits=int(m.group(1)), group_size=group_size, symmetric=m.group(2) == "sym",
                           rounding=rounding, scale_floor=scale_floor)
    raise ConfigError(f"unknown codec name {name!r}")


def int6_flash_pair(group_size: int = 128, rounding: str = "nearest-even") -> tuple[CodecConfig, CodecConfig]:
    """4-bit exchange stage + 8-bit gather stage (codec.py:423-429)."""
    return (CodecConfig(bits=4, group_size=group_size, rounding=rounding),
            CodecConfig(bits=8, group_size=group_size, rounding=rounding))


# --------------------------------------------------------------------------
# tensors


def as_device_tensor(x, device=None) -> torch.Tensor:
    """Flat contiguous CUDA view of `x`; host arrays are copied as float32."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
    if t.dtype not in _TORCH_DTYPES:
        t = t.to(torch.float32)
    if not t.is_cuda:
        t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    return t.reshape(-1).contiguous()


def as_host_tensor(x) -> torch.Tensor:
    """Flat contiguous host view of `x` (torch CPU tensor of a supported dtype,
    else a float32 copy, like as_device_tensor)."""
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float32)))
    if t.dtype not in _TORCH_DTYPES:
        t = t.to(torch.float32)
    return t.reshape(-1).contiguous()


def _stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


class QuantizedTensor:
    """Packed codes plus per-group scale / zero metadata (codec.py:165-219),
    held on the GPU in one device buffer laid out as include/flashcomm.h
    `fc_layout` describes: `codes` (packed uint8, little nibble first),
    `scales_f16` (the fp16 wire scales) and `zeros` (uint8, asymmetric int
    only) are views into it; `scales` is the reference's float32 array.

    The constructor takes the reference's fields, QuantizedTensor(codes,
    scales, zeros, element_count, config) -- numpy arrays, tensors, or a
    packed-bytes object -- and checks them like codec.py:172-181
    (IntegrityError); the library builds instances from device buffers
    (`_from_buffer`)."""

    def __init__(self, codes, scales, zeros, element_count: int, config: CodecConfig, device=None):
        n = int(element_count)
        L = config.device_layout(n)
        groups = config.group_count(n)
        sc = np.asarray(scales.cpu().numpy() if isinstance(scales, torch.Tensor) else scales, dtype=np.float32)
        if sc.shape != (groups,):
            raise IntegrityError(f"expected {groups} scales, got {sc.shape}")
        asym = config.is_int and not config.symmetric
        if asym:
            if zeros is None or np.asarray(zeros.cpu() if isinstance(zeros, torch.Tensor) else zeros).shape != (groups,):
                raise IntegrityError("asymmetric tensor requires one zero per group")
        elif zeros is not None:
            raise IntegrityError("zeros are only present for asymmetric integer codecs")
        raw = codes.data if hasattr(codes, "data") and isinstance(getattr(codes, "data"), (bytes, bytearray)) else codes
        cb = np.frombuffer(bytes(raw), np.uint8) if isinstance(raw, (bytes, bytearray)) else \
            np.asarray(raw.cpu().numpy() if isinstance(raw, torch.Tensor) else raw, dtype=np.uint8).ravel()
        if cb.size != L.codes_bytes:
            raise IntegrityError(f"expected {L.codes_bytes} code bytes, got {cb.size}")
        host = np.zeros(L.total_bytes, np.uint8)
        host[: L.codes_bytes] = cb
        if groups:
            host[L.scales_offset: L.scales_offset + 2 * groups] = sc.astype(np.float16).view(np.uint8)
        if asym:
            z = zeros.cpu().numpy() if isinstance(zeros, torch.Tensor) else zeros
            host[L.zeros_offset: L.zeros_offset + groups] = np.asarray(z, dtype=np.uint8)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._init(torch.from_numpy(host).to(dev), n, config)

    @classmethod
    def _from_buffer(cls, buffer: torch.Tensor, element_count: int, config: CodecConfig) -> "QuantizedTensor":
        q = cls.__new__(cls)
        q._init(buffer, int(element_count), config)
        return q

    def _init(self, buffer: torch.Tensor, element_count: int, config: CodecConfig) -> None:
        self.config = config
        self.element_count = int(element_count)
        self._buf = buffer
        L = config.device_layout(element_count)
        self._layout = L
        self.codes = buffer[: L.codes_bytes]
        if config.is_passthrough:
            self.scales_f16 = torch.empty(0, dtype=torch.float16, device=buffer.device)
        else:
            self.scales_f16 = buffer[L.scales_offset: L.scales_offset + 2 * L.groups].view(torch.float16)
        self.zeros = buffer[L.zeros_offset: L.zeros_offset + L.groups] if (config.is_int and not config.symmetric) else None

    @property
    def scales(self) -> torch.Tensor:
        """float32, one per group (codec.py:168); the wire holds them as fp16 (scales_f16)."""
        return self.scales_f16.float()

    @property
    def group_count(self) -> int:
        return self.config.group_count(self.element_count)

    @property
    def wire_bytes(self) -> int:
        return self.config.wire_byte_len(self.element_count)

    def to_bytes(self) -> bytes:
        """Reference wire format: codes || fp16 scales || zero bytes (codec.py:193-200)."""
        parts = [self.codes.cpu().numpy().tobytes()]
        if self.scales_f16.numel():
            parts.append(self.scales_f16.cpu().numpy().tobytes())
        if self.zeros is not None:
            parts.append(self.zeros.cpu().numpy().tobytes())
        return b"".join(parts)

    @classmethod
    def from_bytes(cls, data: bytes, element_count: int, config: CodecConfig, device=None) -> "QuantizedTensor":
        """Parse a reference wire message (codec.py:202-219) into device layout."""
        expected = config.wire_byte_len(element_count)
        if len(data) != expected:
            raise IntegrityError(f"payload holds {len(data)} bytes, expected {expected}")
        L = config.device_layout(element_count)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        host = np.zeros(L.total_bytes, np.uint8)
        raw = np.frombuffer(data, np.uint8)
        host[: L.codes_bytes] = raw[: L.codes_bytes]
        if not config.is_passthrough:
            g = L.groups
            host[L.scales_offset: L.scales_offset + 2 * g] = raw[L.codes_bytes: L.codes_bytes + 2 * g]
            if config.is_int and not config.symmetric:
                host[L.zeros_offset: L.zeros_offset + g] = raw[L.codes_bytes + 2 * g:]
        return cls._from_buffer(torch.from_numpy(host).to(dev), element_count, config)

    def validate(self) -> None:
        """The reference's decode-time integrity checks (codec.py:360-382):
        scales finite and positive; for integer codecs narrower than their
        storage, every code (the padding nibble of an odd count excluded,
        bitpack.py:64-75) below 2^bits; zero points at most 2^bits - 1. One
        device round trip."""
        cfg = self.config
        if cfg.is_passthrough:
            return
        s = self.scales_f16.float()
        dev = self.codes.device
        bad_scale = (~torch.isfinite(s)).any() | (s <= 0).any()
        bad_code = torch.zeros((), dtype=torch.bool, device=dev)
        bad_zero = torch.zeros((), dtype=torch.bool, device=dev)
        if cfg.is_int and cfg.bits < cfg.storage_bits and self.element_count:
            lim = 1 << cfg.bits
            if cfg.storage_bits == 4:
                lo = self.codes & 0x0F
                hi = self.codes >> 4
                if self.element_count % 2:
                    hi = hi[:-1]
                bad_code = (lo >= lim).any() | (hi >= lim).any()
            else:
                bad_code = (self.codes >= lim).any()
        if cfg.is_int and self.zeros is not None and self.zeros.numel():
            bad_zero = (self.zeros.to(torch.int32) > (1 << cfg.bits) - 1).any()
        flags = torch.stack([bad_scale, bad_code, bad_zero]).cpu().tolist()
        if flags[0]:
            raise IntegrityError("scales must be finite and positive")
        if flags[1]:
            raise IntegrityError(f"code exceeds {cfg.bits}-bit range")
        if flags[2]:
            raise IntegrityError(f"zero point exceeds {cfg.bits}-bit range")


def quantize(x, config: CodecConfig, *, check: bool = True) -> QuantizedTensor:
    """Quantize a flat tensor under `config` (codec.py:292-329) on its GPU.

    check=True synchronizes and raises DomainError for NaN/inf input like the
    reference (codec.py:230-231); check=False leaves the call asynchronous.
    """
    t = as_device_tensor(x)
    n = t.numel()
    if n == 0:
        raise DomainError("input tensor is empty")
    c = config.to_fc()
    L = config.device_layout(n)
    buf = torch.empty(L.total_bytes, dtype=torch.uint8, device=t.device)
    err = torch.zeros(1, dtype=torch.int32, device=t.device) if check else None
    stream = _stream_of(t)
    with torch.cuda.device(t.device):
        _lib.check(_lib.lib().fc_quantize(t.data_ptr(), fc_dtype(t.dtype), n, C.byref(c), buf.data_ptr(),
                                          err.data_ptr() if check else None, stream))
        if check:
            _lib.check(_lib.lib().fc_error_word_check(err.data_ptr(), stream))
    return QuantizedTensor._from_buffer(buf, n, config)


def dequantize(q: QuantizedTensor, dtype: torch.dtype = torch.float32, *, validate: bool = True) -> torch.Tensor:
    """Decode to a flat tensor (codec.py:354-384). float32 output equals the
    reference bit for bit; bf16/fp16 outputs are its RNE rounding.

    Like the reference, the integrity checks run by default and raise
    IntegrityError for corrupt payloads (codec.py:360-382; one device round
    trip). validate=False skips them and keeps the call asynchronous (for
    callers that produced the payload themselves)."""
    if validate:
        q.validate()
    c = q.config.to_fc()
    out = torch.empty(q.element_count, dtype=dtype, device=q._buf.device)
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().fc_dequantize(q._buf.data_ptr(), q.element_count, C.byref(c), out.data_ptr(),
                                            fc_dtype(dtype), _stream_of(out)))
    return out


def group_params_asym(group, bits: int, scale_floor: float = 1e-8) -> tuple[float, int]:
    """Raw (unsnapped) affine parameters of one group (codec.py:251-262):
    scale = max((max - min) / (2^bits - 1), floor), zero = clip(ceil(-min /
    scale), 0, 2^bits - 1), in float64. A tests-only scalar API in the
    reference; the kernels compute the fp16-snapped form (_wire_scale)."""
    if not 2 <= int(bits) <= 8:
        raise DomainError(f"bits must be in 2..8, got {bits}")
    g = _flat_f64(group)
    lo, hi = float(g.min()), float(g.max())
    scale = max((hi - lo) / (2 ** int(bits) - 1), scale_floor)
    zero = int(min(max(np.ceil(np.float64(-lo) / np.float64(scale)), 0), 2 ** int(bits) - 1))
    return float(scale), zero


def group_params_sym(group, bits: int, scale_floor: float = 1e-8) -> float:
    """Raw symmetric scale of one group: max(absmax / (2^(bits-1) - 1), floor)
    (codec.py:265-270)."""
    if not 2 <= int(bits) <= 8:
        raise DomainError(f"bits must be in 2..8, got {bits}")
    g = _flat_f64(group)
    return float(max(float(g.abs().max()) / (2 ** (int(bits) - 1) - 1), scale_floor))


def _flat_f64(x) -> torch.Tensor:
    """float64 flat view, DomainError for empty / non-finite input (codec.py:226-232)."""
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, np.float64))
    t = t.reshape(-1).to(torch.float64)
    if t.numel() == 0:
        raise DomainError("input tensor is empty")
    if not bool(torch.isfinite(t).all()):
        raise DomainError("input contains NaN or infinity")
    return t


def mse(a, b) -> float:
    """Mean squared elementwise difference, float64 (codec.py:387-393)."""
    ta = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, np.float64))
    tb = b if isinstance(b, torch.Tensor) else torch.as_tensor(np.asarray(b, np.float64))
    ta = ta.reshape(-1).to(torch.float64)
    tb = tb.reshape(-1).to(device=ta.device, dtype=torch.float64)
    if ta.numel() != tb.numel():
        raise DomainError(f"length mismatch: {ta.numel()} vs {tb.numel()}")
    if ta.numel() == 0:
        raise DomainError("input tensor is empty")
    return float(torch.mean((ta - tb) ** 2))
