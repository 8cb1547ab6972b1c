"""B200-native Flash All-Reduce (arXiv 2412.04964, "Flash Communication").

Drop-in for the hot path of the reference package `qcollectives`
(/root/reference/pkg/src/qcollectives/__init__.py:3-108): the group codec and
the two-step quantized all-reduce, with the same public names and arguments,
running on hand-written sm_100a kernels behind the C ABI of
include/flashcomm.h (libflashcomm.so).
"""

from .codec import (
    CodecConfig,
    PASSTHROUGH_FP16,
    QuantizedTensor,
    codec_from_name,
    dequantize,
    group_params_asym,
    group_params_sym,
    int6_flash_pair,
    mse,
    quantize,
)
from .collectives import (
    CollectiveRun,
    FlashConfig,
    all_reduce_exact,
    flash_all_reduce,
    run_collective,
    sequential_sum,
)
from .bitpack import magic_dequant_identity, pack, packed_byte_len, unpack
from .comm import FabricTopology, FlashComm, TrafficLedger, flash_ledger
from .errors import ConfigError, CudaError, DomainError, IntegrityError, ProtocolError, QCollectivesError
from .rotation import HadamardBlock, hadamard_apply, hadamard_inverse
from . import tp  # noqa: F401  (registers torch.ops.flashcomm.all_reduce_)

__version__ = "0.1.0"

__all__ = [
    "CodecConfig",
    "CollectiveRun",
    "ConfigError",
    "CudaError",
    "DomainError",
    "FabricTopology",
    "HadamardBlock",
    "FlashComm",
    "FlashConfig",
    "IntegrityError",
    "PASSTHROUGH_FP16",
    "ProtocolError",
    "QCollectivesError",
    "QuantizedTensor",
    "TrafficLedger",
    "all_reduce_exact",
    "codec_from_name",
    "dequantize",
    "flash_all_reduce",
    "flash_ledger",
    "group_params_asym",
    "group_params_sym",
    "magic_dequant_identity",
    "pack",
    "packed_byte_len",
    "unpack",
    "hadamard_apply",
    "hadamard_inverse",
    "int6_flash_pair",
    "mse",
    "quantize",
    "run_collective",
    "sequential_sum",
]
