"""B200 drop-in for ``approx8.codecs`` (reference: pkg/src/approx8/codecs.py).

Same names, argument meaning and error behaviour as the reference codec API
(``DataTypeKind``, ``NormKind``, ``DataTypeSpec``, ``Codebook``,
``build_codebook``, ``QuantizedTensor``, ``encode_buffer``, ``decode_buffer``,
``roundtrip``); the compute runs in the sm_100a kernels of
``include/approx8_b200.h`` on the tensor's CUDA device.  There is no CPU
fallback: without a CUDA device the compute calls raise.

Host and device data:
  * NumPy (or any non-torch) input behaves exactly like the reference:
    ``encode_buffer`` returns a ``QuantizedTensor`` whose ``codes`` is a NumPy
    ``uint8`` array (copied from the GPU on first access; the device copy is
    kept for ``decode_buffer``), and ``decode_buffer`` / ``roundtrip`` /
    ``onebit_decode`` return NumPy ``float32`` arrays; ``OneBitState`` keeps a
    NumPy ``float64`` residual.  The reference's callers (mlp.py:171, 319,
    tensorfile.py:74, cli.py:87-117) run unchanged on it.
  * CUDA tensors stay on the device: ``codes`` is a CUDA ``torch.uint8``
    tensor (flat, C order), decodes return CUDA ``torch.float32`` tensors and
    ``scale`` is a Python float fetched lazily (``scale_tensor`` stays on the
    device, so nothing syncs until it is read).
  * float32 and float64 inputs are encoded exactly as the reference does
    (float64 input through a float64 kernel, codecs.py:254); other dtypes
    are converted to float32 first.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass
from enum import Enum
from functools import lru_cache
from typing import IO, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, InputError, UsageError

SIGN_MASK = 0x80
PAYLOAD_BITS = 7
CODE_COUNT = 256


class DataTypeKind(str, Enum):
    DYNAMIC_TREE = "dynamic-tree"
    STATIC_TREE = "static-tree"
    LINEAR = "linear"
    MANTISSA = "mantissa"


class NormKind(str, Enum):
    NONE = "none"
    ABSMAX = "absmax"
    DECADE = "decade"


# codecs.py:89-94 -- which normalisation fits which codebook family
_ALLOWED_NORMS = {
    DataTypeKind.DYNAMIC_TREE: {NormKind.NONE, NormKind.ABSMAX},
    DataTypeKind.LINEAR: {NormKind.NONE, NormKind.ABSMAX},
    DataTypeKind.STATIC_TREE: {NormKind.NONE, NormKind.DECADE},
    DataTypeKind.MANTISSA: {NormKind.NONE, NormKind.DECADE},
}

DECADE_MIN, DECADE_MAX = -7, 7


@dataclass(frozen=True)
class DataTypeSpec:
    """One concrete codec: a codebook family plus its normalisation
    (codecs.py:99-128, same validation and ``ConfigError`` messages)."""

    kind: DataTypeKind
    normalization: NormKind = NormKind.NONE
    decades: int = 0

    def __post_init__(self) -> None:
        try:
            kind = DataTypeKind(self.kind)
            norm = NormKind(self.normalization)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
        object.__setattr__(self, "kind", kind)
        object.__setattr__(self, "normalization", norm)
        if norm not in _ALLOWED_NORMS[kind]:
            raise ConfigError(f"normalization {norm.value!r} is not supported for {kind.value!r}")
        if norm is NormKind.DECADE:
            if not (DECADE_MIN <= self.decades <= DECADE_MAX):
                raise ConfigError(
                    f"decade offset must lie in [{DECADE_MIN}, {DECADE_MAX}], got {self.decades}"
                )
        elif self.decades != 0:
            raise ConfigError("decades is only meaningful with decade normalization")

    def label(self) -> str:
        if self.normalization is NormKind.DECADE:
            return f"{self.kind.value}/decade{self.decades:+d}"
        return f"{self.kind.value}/{self.normalization.value}"

    # codes used by the C ABI
    @property
    def kind_code(self) -> int:
        return N.KIND_CODE[self.kind.value]

    @property
    def norm_code(self) -> int:
        return N.NORM_CODE[self.normalization.value]


def parse_spec(label: str) -> DataTypeSpec:
    """Inverse of ``DataTypeSpec.label`` ("dynamic-tree/absmax", "mantissa/decade+2")."""
    kind, _, norm = label.partition("/")
    norm = norm or "none"
    if norm.startswith("decade"):
        return DataTypeSpec(DataTypeKind(kind), NormKind.DECADE, int(norm[6:] or 0))
    return DataTypeSpec(DataTypeKind(kind), NormKind(norm))


# ---------------------------------------------------------------------------
# codebooks


_dev_lock = threading.Lock()
_dev_cache: dict = {}


@dataclass(frozen=True, eq=False)
class Codebook:
    """Decode table for all 256 codes plus the encode search structures
    (codecs.py:161-183).  Host arrays are read-only NumPy views; the device
    copies (table struct, fixed-scale decision table) are built lazily per
    CUDA device."""

    spec: DataTypeSpec
    decode_table: np.ndarray
    sorted_values: np.ndarray
    sorted_codes: np.ndarray
    _book: N.Book = None  # type: ignore[assignment]

    @property
    def zero_code(self) -> int:
        return int(self.sorted_codes[0])

    def dump(self, out: IO[str]) -> None:
        """Write all 256 codes as 'code<TAB>value' lines (codecs.py:180-183)."""
        for code in range(CODE_COUNT):
            out.write(f"0x{code:02x}\t{self.decode_table[code]:.9g}\n")

    @property
    def fixed_scale(self) -> Optional[float]:
        """The data-independent scale of none/decade specs (codecs.py:232-241)."""
        if self.spec.normalization is NormKind.ABSMAX:
            return None
        s = C.c_float()
        N.check(N.lib.a8_fixed_scale(self.spec.norm_code, int(self.spec.decades), C.byref(s)))
        return float(s.value)

    def device_tables(self, device: torch.device):
        """(book struct bytes, fixed-scale decision table or None) on ``device``."""
        dev = _cuda_device(device)
        key = (self.spec, dev.index)
        with _dev_lock:
            hit = _dev_cache.get(key)
            if hit is None:
                book = torch.frombuffer(bytearray(bytes(self._book)), dtype=torch.uint8).to(dev)
                lut = None
                if self.spec.normalization is not NormKind.ABSMAX:
                    host = N.Lut()
                    N.check(N.lib.a8_build_lut_host(C.byref(self._book), self.fixed_scale, C.byref(host)))
                    lut = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
                hit = (book, lut)
                _dev_cache[key] = hit
        return hit


@lru_cache(maxsize=None)
def build_codebook(spec: DataTypeSpec) -> Codebook:
    """codecs.py:186-204, computed by the library's host builder (a8_codebook)."""
    book = N.Book()
    N.check(N.lib.a8_codebook(spec.kind_code, C.byref(book)))
    d = int(book.ndistinct)
    table = np.frombuffer(bytes(book.table), dtype=np.float32).copy()
    values = np.frombuffer(bytes(book.values), dtype=np.float64)[:d].copy()
    codes = np.frombuffer(bytes(book.codes), dtype=np.uint8)[:d].copy()
    for arr in (table, values, codes):
        arr.setflags(write=False)
    return Codebook(spec=spec, decode_table=table, sorted_values=values, sorted_codes=codes, _book=book)


# ---------------------------------------------------------------------------
# quantized tensors


class QuantizedTensor:
    """Encoded buffer plus everything needed to decode it (codecs.py:207-229).

    ``codes``  uint8, one byte per element, flat C order: a CUDA tensor for
               device input, a NumPy array for host input (materialised from
               the device copy on first access; once exposed, the NumPy array
               is what decodes read, so in-place edits are honoured)
    ``scale``  float32 normalisation scale as a Python float (lazy)
    """

    def __init__(
        self,
        codes,
        shape: Sequence[int],
        spec: Optional[DataTypeSpec],
        scale: Optional[float] = None,
        nbits: int = 8,
        pos_level: float = 0.0,
        neg_level: float = 0.0,
        *,
        scale_tensor: Optional[torch.Tensor] = None,
        meta: Optional[torch.Tensor] = None,
    ) -> None:
        self._dev_codes: Optional[torch.Tensor] = None
        self._np_codes: Optional[np.ndarray] = None
        self._host = False
        self.codes = codes
        self.shape = tuple(int(d) for d in shape)
        self.spec = spec
        self.nbits = nbits
        self._levels = (pos_level, neg_level)
        self.levels_tensor: Optional[torch.Tensor] = None  # device float[2] (1-bit tensors)
        self._scale = None if scale is None else float(np.float32(scale))
        self.scale_tensor = scale_tensor
        self._meta = meta  # int32[2] = [status, scale bits] written by the encoder
        self._checked = meta is None
        self.block_size: Optional[int] = None  # per-block scales (encode_buffer(block_size=...))
        self.block_scales: Optional[torch.Tensor] = None
        self._block_status: Optional[torch.Tensor] = None

    @property
    def codes(self):
        if self._np_codes is not None:
            return self._np_codes
        if self._host and self._dev_codes is not None:
            self._np_codes = self._dev_codes.cpu().numpy()  # host caller: the reference's ndarray
        return self._np_codes if self._host else self._dev_codes

    @codes.setter
    def codes(self, c) -> None:
        if isinstance(c, torch.Tensor):
            self._dev_codes, self._np_codes, self._host = c, None, False
        else:
            self._dev_codes, self._np_codes, self._host = None, np.asarray(c), True

    def _set_device_result(self, codes: torch.Tensor, host: bool) -> "QuantizedTensor":
        """Codes produced on the device for a host (NumPy) or device caller."""
        self._dev_codes, self._np_codes, self._host = codes, None, bool(host)
        return self

    @property
    def is_host(self) -> bool:
        """True when the tensor came from (and decodes to) host NumPy data."""
        return self._host

    def _host_levels(self):
        if self.levels_tensor is not None and self._levels is None:
            lv = self.levels_tensor.cpu()
            self._levels = (float(lv[0]), float(lv[1]))
        return self._levels

    @property
    def pos_level(self) -> float:
        return self._host_levels()[0]

    @pos_level.setter
    def pos_level(self, v: float) -> None:
        self._levels = (float(v), self._host_levels()[1])
        self.levels_tensor = None

    @property
    def neg_level(self) -> float:
        return self._host_levels()[1]

    @neg_level.setter
    def neg_level(self, v: float) -> None:
        self._levels = (self._host_levels()[0], float(v))
        self.levels_tensor = None

    @property
    def count(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def scale(self) -> float:
        if self.block_size is not None:
            raise UsageError("this tensor has one scale per block: use block_scales")
        if self._scale is None:
            self._finish()
        return self._scale

    @scale.setter
    def scale(self, value: float) -> None:
        self._scale = float(np.float32(value))
        self.scale_tensor = None

    def _finish(self) -> None:
        """Sync on the encoder's status word; raise InputError for NaN/Inf
        input exactly where the reference does (codecs.py:251-252)."""
        if self._block_status is not None:
            st = int(self._block_status.cpu()[0])
            self._block_status = None
            if st & N.A8_STATUS_NONFINITE:
                raise InputError("cannot encode non-finite values (NaN or Inf present)")
            return
        if self._checked and self._scale is not None:
            return
        if self._meta is not None:
            host = self._meta.cpu()
            status = int(host[0])
            if status & N.A8_STATUS_AMAX_MISMATCH:
                raise UsageError("the supplied amax is not max|x| of the input")
            if status & N.A8_STATUS_NONFINITE:
                raise InputError("cannot encode non-finite values (NaN or Inf present)")
            self._scale = float(host[1:].view(torch.float32)[0])
            self._checked = True
        elif self.scale_tensor is not None:
            self._scale = float(self.scale_tensor.float().cpu()[0])

    def device_codes(self, device: torch.device) -> torch.Tensor:
        c = self._np_codes if self._np_codes is not None else self._dev_codes
        if not isinstance(c, torch.Tensor):
            c = torch.from_numpy(np.ascontiguousarray(np.asarray(c, dtype=np.uint8).ravel()))
        c = c.to(device).reshape(-1)
        if not c.is_contiguous() or c.data_ptr() % 16:
            c = c.clone()
        return c

    def device_scale(self, device: torch.device) -> torch.Tensor:
        if self.scale_tensor is not None and self.scale_tensor.device == device:
            return self.scale_tensor
        return torch.tensor([self.scale], dtype=torch.float32, device=device)

    def codes_numpy(self) -> np.ndarray:
        c = self.codes
        return c.cpu().numpy() if isinstance(c, torch.Tensor) else np.asarray(c, dtype=np.uint8)

    @property
    def codes_device(self) -> Optional[torch.Tensor]:
        """The CUDA copy of the codes, if there is one (None for codes that
        only exist on the host)."""
        return self._dev_codes

    def __repr__(self) -> str:
        label = self.spec.label() if self.spec is not None else None
        return f"QuantizedTensor(shape={self.shape}, spec={label}, nbits={self.nbits})"


# ---------------------------------------------------------------------------
# device plumbing


def _cuda_device(device) -> torch.device:
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise UsageError(f"the approx8 B200 codec runs on CUDA devices only, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


_ws_lock = threading.Lock()
_ws_cache: dict = {}
# Minimum capacity: every call of <= 32 segments (all graph-capturable calls)
# shares the first allocation, so a captured graph's workspace pointer stays
# valid; a larger call reallocates and bumps the epoch (see workspace_epoch).
WS_MIN_SEGS = 32
_ws_epoch: dict = {}


def workspace(device: torch.device, stream: int, nseg: int) -> torch.Tensor:
    """Zero-filled kernel scratch for (device, stream); the kernels leave it
    zeroed, so it is allocated once and grown on demand."""
    need = N.workspace_bytes(max(nseg, WS_MIN_SEGS))
    key = (device.index, stream)
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(need, dtype=torch.uint8, device=device)
            _ws_cache[key] = ws
            _ws_epoch[key] = _ws_epoch.get(key, 0) + 1
    return ws


def workspace_epoch(device: torch.device, stream: int) -> int:
    """Bumped whenever ``workspace(device, stream, ...)`` reallocates: a CUDA
    graph captured under an older epoch holds a freed workspace address."""
    with _ws_lock:
        return _ws_epoch.get((device.index, stream), 0)


def as_device_f32(x, device=None) -> tuple[torch.Tensor, tuple]:
    """Input to a contiguous float32 CUDA tensor (H2D copy for host data)."""
    if isinstance(x, torch.Tensor):
        dev = _cuda_device(x.device if x.is_cuda else device)
        t = x
        if t.dtype != torch.float32:
            t = t.to(torch.float32)
        t = t.to(dev, non_blocking=True).contiguous()
        return t, tuple(x.shape)
    arr = np.asarray(x)
    shape = tuple(arr.shape)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float32)
    dev = _cuda_device(device)
    t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(dev)
    return t, shape


def round16(n: int) -> int:
    return (int(n) + 15) // 16 * 16


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


# ---------------------------------------------------------------------------
# codec entry points


BLOCK_SIZES = (1024, 2048, 4096)


def encode_buffer(x, codebook: Codebook, *, device=None, sync: bool = True,
                  block_size: Optional[int] = None, amax=None) -> QuantizedTensor:
    """Quantise ``x`` to the nearest codebook values (codecs.py:244-269).

    Ties go to the smaller magnitude; the sign bit is set only on non-zero
    values; non-finite input raises ``InputError``.  With ``sync=False`` the
    call is fully asynchronous and the check happens when ``scale`` is read.

    ``block_size`` (1024, 2048 or 4096; absmax specs only) selects per-block
    scales: every block of that many consecutive elements is encoded exactly
    as ``encode_buffer`` would encode it alone (its own absmax).  The scales
    are ``q.block_scales``.  Not a reference feature (the north star's
    optional per-block max-abs); single pass on the GPU.

    ``amax`` (absmax specs, CUDA input): a float32 device tensor holding
    max|x|, written by the kernel that produced x (``relu_absmax``,
    ``scale_absmax_``): the encode skips its max pass (a8_encode_premax).
    A value that is not max|x| raises UsageError.
    """
    spec = codebook.spec
    if amax is not None:
        if (spec.normalization is not NormKind.ABSMAX or block_size is not None
                or not isinstance(x, torch.Tensor) or x.dtype != torch.float32 or not x.is_cuda):
            raise UsageError("amax needs an absmax spec and a float32 CUDA tensor (no block_size)")
        if (not isinstance(amax, torch.Tensor) or amax.dtype != torch.float32 or amax.numel() != 1
                or amax.device != x.device):
            raise UsageError("amax must be a 1-element float32 tensor on the input's device")
    if block_size is not None:
        return _encode_blocked(x, codebook, device, sync, int(block_size))
    if _is_f64(x):  # the reference computes float64 input in float64 (codecs.py:254)
        return _encode_f64(x, codebook, device, sync)
    host = not isinstance(x, torch.Tensor)
    t, shape = as_device_f32(x, device)
    dev = t.device
    n = t.numel()
    if n == 0:  # codecs.py:257-258
        s = codebook.fixed_scale
        return QuantizedTensor(torch.empty(0, dtype=torch.uint8, device=dev), shape, spec,
                               1.0 if s is None else s)._set_device_result(
                                   torch.empty(0, dtype=torch.uint8, device=dev), host)
    book, lut = codebook.device_tables(dev)
    with torch.cuda.device(dev):
        stream = _stream(dev)
        meta = torch.empty(2, dtype=torch.int32, device=dev)  # both words written by the kernel
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        seg = N.EncSeg(t.data_ptr(), n, 0, 0, 0)
        lay = N.Layout(codes.data_ptr(), meta.data_ptr() + 4, round16(n), round16(n), 0, 0, 1, 0)
        ws = workspace(dev, stream, 1)
        if amax is not None:
            N.check(N.lib.a8_encode_premax(C.byref(seg), 1, book.data_ptr(), amax.data_ptr(), lay, ws.data_ptr(),
                                           ws.numel(), None, meta.data_ptr(), stream))
        else:
            N.check(N.lib.a8_encode(C.byref(seg), 1, book.data_ptr(), spec.norm_code,
                                    None if lut is None else lut.data_ptr(), lay, ws.data_ptr(),
                                    ws.numel(), None, meta.data_ptr(), stream))
    q = QuantizedTensor(codes, shape, spec, scale_tensor=meta[1:].view(torch.float32), meta=meta)
    q._set_device_result(codes, host)
    q._keepalive = t  # input must outlive the asynchronous kernel
    if sync:
        q._finish()
    return q


def _encode_blocked(x, codebook: Codebook, device, sync: bool, block: int) -> QuantizedTensor:
    spec = codebook.spec
    if spec.normalization is not NormKind.ABSMAX:
        raise ConfigError(f"per-block scales need absmax normalization, not {spec.normalization.value!r}")
    if block not in BLOCK_SIZES:
        raise ConfigError(f"block_size must be one of {BLOCK_SIZES}, got {block}")
    host = not isinstance(x, torch.Tensor)
    t, shape = as_device_f32(x, device)
    t = t.reshape(-1)
    dev = t.device
    n = t.numel()
    nblk = -(-n // block)
    book, _ = codebook.device_tables(dev)
    with torch.cuda.device(dev):
        stream = _stream(dev)
        codes = torch.empty(max(n, 4), dtype=torch.uint8, device=dev)[:n]
        scales = torch.empty(max(nblk, 1), dtype=torch.float32, device=dev)[:nblk]
        status = torch.empty(1, dtype=torch.int32, device=dev)
        N.check(N.lib.a8_encode_blocked(t.data_ptr(), n, block, book.data_ptr(), codes.data_ptr(),
                                        scales.data_ptr(), status.data_ptr(), stream))
    q = QuantizedTensor(codes, shape, spec, 1.0, scale_tensor=None)._set_device_result(codes, host)
    q.block_size = block
    q.block_scales = scales
    q._block_status = status
    q._keepalive = t
    if sync:
        q._finish()
    return q


def _is_f64(x) -> bool:
    if isinstance(x, torch.Tensor):
        return x.dtype == torch.float64
    return np.asarray(x).dtype == np.float64


def _encode_f64(x, codebook: Codebook, device, sync: bool) -> QuantizedTensor:
    """float64 input: the reference decision restated in float64 on the GPU
    (a8_encode_f64), bit-exact with codecs.py:254-268 for any float64 data."""
    spec = codebook.spec
    host = not isinstance(x, torch.Tensor)
    if isinstance(x, torch.Tensor):
        dev = _cuda_device(x.device if x.is_cuda else device)
        shape = tuple(x.shape)
        t = x.to(dev).contiguous().reshape(-1)
    else:
        arr = np.asarray(x)
        shape = tuple(arr.shape)
        dev = _cuda_device(device)
        t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).to(dev)
    n = t.numel()
    if n == 0:
        s = codebook.fixed_scale
        e = torch.empty(0, dtype=torch.uint8, device=dev)
        return QuantizedTensor(e, shape, spec, 1.0 if s is None else s)._set_device_result(e, host)
    book, _ = codebook.device_tables(dev)
    fixed = codebook.fixed_scale
    with torch.cuda.device(dev):
        stream = _stream(dev)
        meta = torch.empty(2, dtype=torch.int32, device=dev)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        seg = N.EncSeg64(t.data_ptr(), n, 0, 0, 0)
        lay = N.Layout(codes.data_ptr(), meta.data_ptr() + 4, round16(n), round16(n), 0, 0, 1, 0)
        ws = workspace(dev, stream, 1)
        N.check(N.lib.a8_encode_f64(C.byref(seg), 1, book.data_ptr(), spec.norm_code,
                                    1.0 if fixed is None else fixed, lay, ws.data_ptr(), ws.numel(),
                                    None, meta.data_ptr(), stream))
    q = QuantizedTensor(codes, shape, spec, scale_tensor=meta[1:].view(torch.float32), meta=meta)
    q._set_device_result(codes, host)
    q._keepalive = t
    if sync:
        q._finish()
    return q


def decode_buffer(q: QuantizedTensor, codebook: Codebook, *, device=None, out=None):
    """Map codes back to float32 values, undoing the scale (codecs.py:272-282).

    Returns a CUDA float32 tensor, or a NumPy float32 array of ``q.shape``
    when ``q`` holds host (NumPy) data, as the reference does."""
    y = _decode_device(q, codebook, device, out)
    if q.is_host and out is None:
        return y.cpu().numpy()
    return y


def _decode_device(q: QuantizedTensor, codebook: Codebook, device, out) -> torch.Tensor:
    if q.nbits != 8:
        raise UsageError("decode_buffer handles 8-bit tensors; use onebit_decode")
    if q.spec != codebook.spec:
        raise UsageError(
            f"tensor was encoded as {q.spec and q.spec.label()}, codebook is {codebook.spec.label()}"
        )
    dc = q.codes_device
    if dc is not None and dc.is_cuda and q._np_codes is None:
        dev = dc.device
    else:
        dev = _cuda_device(device)
    codes = q.device_codes(dev)
    n = codes.numel()
    if n != q.count:
        raise UsageError(f"codes hold {n} elements, shape {q.shape} needs {q.count}")
    if out is None:
        out = torch.empty(q.shape, dtype=torch.float32, device=dev)
    elif out.dtype != torch.float32 or not out.is_contiguous() or out.numel() != n or out.device != dev:
        raise UsageError("out must be a contiguous float32 tensor of the decoded size on the codes' device")
    if n == 0:
        return out
    book, _ = codebook.device_tables(dev)
    if q.block_size is not None:
        with torch.cuda.device(dev):
            if codes.data_ptr() % 4:
                codes = codes.clone()
            sc = q.block_scales.to(dev).contiguous()
            N.check(N.lib.a8_decode_blocked(codes.data_ptr(), n, q.block_size, sc.data_ptr(), book.data_ptr(),
                                            out.data_ptr(), _stream(dev)))
        return out
    with torch.cuda.device(dev):
        stream = _stream(dev)
        scale_t = q.device_scale(dev)
        seg = N.DecSeg(out.data_ptr(), n, 0, 0, 0)
        lay = N.Layout(codes.data_ptr(), scale_t.data_ptr(), round16(n), round16(n), 0, 0, 1, 0)
        ws = workspace(dev, stream, 1)
        N.check(N.lib.a8_decode(C.byref(seg), 1, book.data_ptr(), lay, 1, 0, -1, 0, None,
                                ws.data_ptr(), ws.numel(), stream))
    return out


def _roundtrip_fused(t: torch.Tensor, codebook: Codebook) -> Optional[torch.Tensor]:
    """decode(encode(t)) in one kernel (a8_roundtrip) when the call fits in
    the GPU's shared memory; None otherwise.  t: contiguous float32 CUDA."""
    dev = t.device
    n = t.numel()
    if n == 0 or n > RESIDENT_MAX_ELEMS:
        return None
    book, lut = codebook.device_tables(dev)
    out = torch.empty_like(t)
    with torch.cuda.device(dev):
        stream = _stream(dev)
        meta = torch.empty(2, dtype=torch.int32, device=dev)  # [status, scale]
        seg = N.EncSeg(t.data_ptr(), n, 0, 0, 0)
        outs = (C.c_void_p * 1)(out.data_ptr())
        ws = workspace(dev, stream, 1)
        rc = N.lib.a8_roundtrip(C.byref(seg), outs, 1, book.data_ptr(), codebook.spec.norm_code,
                                None if lut is None else lut.data_ptr(), meta.data_ptr() + 4, meta.data_ptr(),
                                ws.data_ptr(), ws.numel(), stream)
    if rc == N.A8_ERR_USAGE:
        return None
    N.check(rc)
    if int(meta[0].cpu()) & N.A8_STATUS_NONFINITE:  # codecs.py:251-252
        raise InputError("cannot encode non-finite values (NaN or Inf present)")
    return out


# largest single call the fused round trip takes (148 SMs x 51196 elements)
RESIDENT_MAX_ELEMS = 148 * 51196


def roundtrip(x, spec: DataTypeSpec, *, device=None):
    """encode + decode in one step (codecs.py:285-288).  NumPy in -> NumPy out.

    float32 data that fits in the GPU's shared memory takes one fused kernel
    (the codes are never stored); anything else runs encode then decode."""
    cb = build_codebook(spec)
    if not _is_f64(x):
        t, shape = as_device_f32(x, device)
        y = _roundtrip_fused(t.reshape(-1), cb)
        if y is not None:
            y = y.reshape(shape)
            return y if isinstance(x, torch.Tensor) else y.cpu().numpy()
    q = encode_buffer(x, cb, device=device, sync=False)
    y = _decode_device(q, cb, device, None)
    q._finish()
    if isinstance(x, torch.Tensor):
        return y
    return y.cpu().numpy()


# ---------------------------------------------------------------------------
# 1-bit quantizer with error feedback (codecs.py:291-348)


class OneBitState:
    """Residual carried between successive 1-bit quantizations of one tensor
    (codecs.py:295-303).  ``residual`` is a NumPy float64 array for host
    callers (the reference's type; ``onebit_quantize`` rebinds it to a new
    array, as codecs.py:335 does) or a float64 CUDA tensor for a
    device-resident state (updated in place, no host traffic)."""

    def __init__(self, residual) -> None:
        self.residual = residual

    @classmethod
    def zeros(cls, shape, device=None) -> "OneBitState":
        shp = (shape,) if isinstance(shape, int) else tuple(shape)
        if device is None:
            return cls(np.zeros(shp, dtype=np.float64))
        return cls(torch.zeros(shp, dtype=torch.float64, device=_cuda_device(device)))


_ob_ws: dict = {}

_NONFINITE_MSG = "cannot encode non-finite values (NaN or Inf present)"


def onebit_quantize(g, state: OneBitState, *, sync: bool = True, device=None) -> QuantizedTensor:
    """Quantize ``g + residual`` to one bit per element and update ``state``
    (codecs.py:306-339): each side of 0 is reconstructed as its own float32
    mean and the residual keeps exactly what the receiver cannot see.

    Non-finite input raises ``InputError`` and leaves the state untouched
    (codecs.py:317-318).  A host state (NumPy residual) is always checked
    before returning; a device state with ``sync=False`` is checked by
    ``q._finish()``."""
    res = state.residual
    host = not isinstance(res, torch.Tensor)
    if host:
        res_np = np.asarray(res, dtype=np.float64)
        gdev = g.device if isinstance(g, torch.Tensor) and g.is_cuda else device
        dev = _cuda_device(gdev)
        res_shape = tuple(res_np.shape)
    else:
        if not res.is_cuda or res.dtype != torch.float64:
            state.residual = res = res.to(device=_cuda_device(device if not res.is_cuda else res.device),
                                          dtype=torch.float64)
        dev = res.device
        res_shape = tuple(res.shape)
    if isinstance(g, torch.Tensor):
        shape = tuple(g.shape)
        t = g.to(dev)
    else:
        arr = np.asarray(g)
        shape = tuple(arr.shape)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    if shape != res_shape:
        raise UsageError(f"gradient shape {shape} does not match residual shape {res_shape}")
    if t.dtype not in (torch.float32, torch.float64):  # float32 widens exactly; the rest as np.asarray(g, float64)
        t = t.to(torch.float64)
    t = t.contiguous()
    if host:
        res_c = torch.from_numpy(np.ascontiguousarray(res_np).copy()).to(dev)
    else:
        res_c = res if res.is_contiguous() else res.contiguous()
    n = t.numel()
    bits = torch.empty((n + 7) // 8, dtype=torch.uint8, device=dev)
    lv = torch.zeros(2, dtype=torch.float32, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = None
    if n:
        with torch.cuda.device(dev):
            ws = _ob_ws.get(dev.index)
            if ws is None:
                ws = _ob_ws[dev.index] = torch.empty(N.lib.a8_onebit_workspace_bytes(), dtype=torch.uint8,
                                                     device=dev)
            N.check(N.lib.a8_onebit_quantize(t.data_ptr(), 1 if t.dtype == torch.float64 else 0, res_c.data_ptr(),
                                             n, bits.data_ptr(), lv.data_ptr(), status.data_ptr(), ws.data_ptr(),
                                             ws.numel(), _stream(dev)))
    if host:
        if n and int(status.cpu()[0]) & N.A8_STATUS_NONFINITE:
            raise InputError(_NONFINITE_MSG)
        lvh = lv.cpu()
        state.residual = res_c.cpu().numpy().reshape(res_shape)
        return QuantizedTensor(bits.cpu().numpy(), shape, None, 1.0, nbits=1,
                               pos_level=float(lvh[0]), neg_level=float(lvh[1]))
    if res_c is not res:
        res.copy_(res_c)
    q = QuantizedTensor(bits, shape, None, 1.0, nbits=1)
    q._levels = None
    q.levels_tensor = lv
    q._keepalive = (t, ws)
    if n:
        q._block_status = status
    if sync:
        q._finish()
    return q


def onebit_decode(q: QuantizedTensor, *, device=None):
    """Reconstruct the two-level float32 tensor (codecs.py:342-348): a CUDA
    tensor, or a NumPy array when ``q`` holds host data."""
    if q.nbits != 1:
        raise UsageError("onebit_decode expects a 1-bit tensor")
    dc = q.codes_device
    dev = dc.device if dc is not None and dc.is_cuda and q._np_codes is None else _cuda_device(device)
    codes = q.device_codes(dev)
    n = q.count
    lv = q.levels_tensor if q.levels_tensor is not None else torch.tensor(
        [np.float32(q.pos_level), np.float32(q.neg_level)], dtype=torch.float32, device=dev)
    out = torch.empty(q.shape, dtype=torch.float32, device=dev)
    if n:
        with torch.cuda.device(dev):
            N.check(N.lib.a8_onebit_decode(codes.data_ptr(), n, lv.data_ptr(), out.data_ptr(), _stream(dev)))
    return out.cpu().numpy() if q.is_host else out
