"""ctypes binding of libflashcomm.so (the C ABI in include/flashcomm.h).

The library is built in-tree by `__graft_entry__.build()` /
`make -C paper_2412_04964_b200/csrc`. There is no fallback: every compute
entry point of this package goes through this library, and a missing
library raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import STATUS_TO_ERROR, CudaError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libflashcomm.so")

FC_MAX_RANKS = 16
FC_IPC_HANDLE_BYTES = 64

DTYPE_F32, DTYPE_F16, DTYPE_BF16 = 0, 1, 2
KIND_INT, KIND_FP16, KIND_MINIFLOAT = 0, 1, 2
MINIFLOAT_FORMAT_IDS = {"e4m3": 0, "e5m2": 1, "e2m1": 2}
ROUND_NEAREST_EVEN, ROUND_CEIL = 0, 1
OPT_FUSED, OPT_CTAS, OPT_TIMEOUT_MS, OPT_LAG, OPT_FAST, OPT_LAST_LAUNCHES, OPT_REDUCE_STAGES = 0, 1, 2, 3, 4, 5, 6
OPT_SCATTER_STAGES, OPT_GATHER_STAGES, OPT_CTAS_PER_SM, OPT_STREAM_MASK, OPT_PHASES = 7, 8, 9, 10, 11
OPT_FUSED_CHUNK, OPT_ONESHOT, OPT_HOST_CHUNK_BYTES, OPT_FUSED_GATHER_CTAS, OPT_ROLE_PROFILE = 12, 13, 14, 15, 16


class fc_codec(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("bits", C.c_int32),
        ("group_size", C.c_int32),
        ("symmetric", C.c_int32),
        ("rounding", C.c_int32),
        ("reserved", C.c_int32),
        ("scale_floor", C.c_double),
    ]


class fc_flash_cfg(C.Structure):
    _fields_ = [("stage1", fc_codec), ("stage2", fc_codec), ("chunk_elems", C.c_int64)]


class fc_layout(C.Structure):
    _fields_ = [
        ("elements", C.c_int64),
        ("groups", C.c_int64),
        ("codes_bytes", C.c_int64),
        ("scales_offset", C.c_int64),
        ("zeros_offset", C.c_int64),
        ("total_bytes", C.c_int64),
        ("wire_bytes", C.c_int64),
    ]


_P = C.c_void_p
_I32, _I64 = C.c_int32, C.c_int64
_SIGS = {
    "fc_version": (C.c_char_p, []),
    "fc_last_error": (C.c_char_p, []),
    "fc_codec_validate": (C.c_int, [C.POINTER(fc_codec)]),
    "fc_codec_layout": (C.c_int, [C.POINTER(fc_codec), _I64, C.POINTER(fc_layout)]),
    "fc_flash_resolve_chunk": (C.c_int, [C.POINTER(fc_flash_cfg), _I32, C.POINTER(_I64)]),
    "fc_quantize": (C.c_int, [_P, _I32, _I64, C.POINTER(fc_codec), _P, _P, _P]),
    "fc_dequantize": (C.c_int, [_P, _I64, C.POINTER(fc_codec), _P, _I32, _P]),
    "fc_error_word_check": (C.c_int, [_P, _P]),
    "fc_comm_create_local": (C.c_int, [_I32, C.POINTER(_I32), _I64, C.POINTER(_P)]),
    "fc_comm_create_ipc": (C.c_int, [_I32, _I32, _I32, _I64, C.POINTER(_P)]),
    "fc_comm_ipc_handle": (C.c_int, [_P, _P]),
    "fc_comm_ipc_open": (C.c_int, [_P, _P]),
    "fc_comm_destroy": (C.c_int, [_P]),
    "fc_comm_set_option": (C.c_int, [_P, _I32, _I64]),
    "fc_comm_get_option": (C.c_int, [_P, _I32, C.POINTER(_I64)]),
    "fc_flash_all_reduce_local": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), _I64, _I32, _I32,
                                            C.POINTER(fc_flash_cfg), C.POINTER(_P)]),
    "fc_flash_all_reduce_host": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), _I64, _I32, _I32,
                                           C.POINTER(fc_flash_cfg)]),
    "fc_flash_all_reduce_host_rank": (C.c_int, [_P, _P, _P, _I64, _I32, _I32, C.POINTER(fc_flash_cfg)]),
    "fc_flash_all_reduce": (C.c_int, [_P, _P, _P, _I64, _I32, _I32, C.POINTER(fc_flash_cfg), _P]),
    "fc_comm_check": (C.c_int, [_P, _I32]),
    "fc_comm_teardown_check": (C.c_int, [_P]),
    "fc_comm_slot": (C.c_int, [_P, _I32, _I32, _I32, _P, C.POINTER(fc_layout)]),
    "fc_comm_topology": (C.c_int, [_P, C.POINTER(_I32), C.POINTER(_I32)]),
    "fc_comm_role_profile": (C.c_int, [_P, _I32, C.POINTER(C.c_uint64), _I32, C.POINTER(_I32)]),
    "fc_hadamard": (C.c_int, [_P, _I32, _I64, _I64, _I32, _I32, _P, _I32, _P, _I32, _I64, _P]),
    "fc_comm_set_rotation": (C.c_int, [_P, _I32, _I32, _I32, _P]),
    "fc_flash_rotation_fusable": (_I32, [_P, _I64, C.POINTER(fc_flash_cfg), _I32]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load libflashcomm.so once; raise loudly when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libflashcomm.so not found at {LIB_PATH}: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` or "
                    "`make -C paper_2412_04964_b200/csrc` (no CPU fallback exists)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int) -> None:
    """Map an fc_status to the reference exception taxonomy."""
    if status == 0:
        return
    msg = lib().fc_last_error().decode(errors="replace")
    raise STATUS_TO_ERROR.get(int(status), CudaError)(msg)
