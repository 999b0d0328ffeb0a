"""B200-native 8-bit approximation hot path (arXiv 1511.04561), drop-in for the
codec / exchange subset of the reference package ``approx8``
(``approx8/__init__.py:9-22`` codec re-exports, ``mlp.py`` hook seams).

Compute runs in hand-written sm_100a kernels behind the C ABI declared in
``include/approx8_b200.h``; the Python layer mirrors the reference API.
"""

from .codecs import (
    CODE_COUNT,
    PAYLOAD_BITS,
    SIGN_MASK,
    Codebook,
    DataTypeKind,
    DataTypeSpec,
    NormKind,
    OneBitState,
    QuantizedTensor,
    build_codebook,
    decode_buffer,
    encode_buffer,
    onebit_decode,
    onebit_quantize,
    parse_spec,
    roundtrip,
)
from .errorbench import ErrorReport, SampleSpec, measure_error, run_error_suite
from .errors import ApproxError, ConfigError, InputError, TrainingError, UsageError
from .exchange import (
    ONEBIT,
    CompressedAllGather,
    DDPHookState,
    GradientExchange,
    LocalExchange,
    OneBitExchange,
    PeerExchange,
    PeerTransport,
    SymmetricMemoryTransport,
    a8_comm_hook,
    exchange,
)
from .produce import relu_absmax, scale_absmax_
from .tensorfile import read_tensor, write_tensor
from .hooks import (
    HookMode,
    HookStats,
    ModelParallelFC,
    QuantHookConfig,
    default_hook_spec,
    make_quantizer,
)

__all__ = [
    "CODE_COUNT",
    "PAYLOAD_BITS",
    "SIGN_MASK",
    "ApproxError",
    "Codebook",
    "CompressedAllGather",
    "ConfigError",
    "DDPHookState",
    "DataTypeKind",
    "DataTypeSpec",
    "ErrorReport",
    "GradientExchange",
    "OneBitExchange",
    "PeerExchange",
    "PeerTransport",
    "SymmetricMemoryTransport",
    "ONEBIT",
    "HookMode",
    "HookStats",
    "InputError",
    "LocalExchange",
    "ModelParallelFC",
    "NormKind",
    "OneBitState",
    "QuantHookConfig",
    "QuantizedTensor",
    "SampleSpec",
    "TrainingError",
    "UsageError",
    "a8_comm_hook",
    "build_codebook",
    "decode_buffer",
    "default_hook_spec",
    "encode_buffer",
    "exchange",
    "make_quantizer",
    "measure_error",
    "onebit_decode",
    "onebit_quantize",
    "parse_spec",
    "read_tensor",
    "relu_absmax",
    "roundtrip",
    "run_error_suite",
    "scale_absmax_",
    "write_tensor",
]
