"""Hook-seam configuration and GPU seams (reference: approx8/mlp.py).

``HookMode``, ``QuantHookConfig`` and ``default_hook_spec`` keep the names,
defaults and validation of mlp.py:90-121 and mlp.py:399-411.  The seams are
the places where a tensor crosses a device boundary:

  * data parallel (mlp.py:367-369): every W/b gradient -> ``GradientExchange``
    (8-bit all-gather + fused decode-average) instead of an fp32 all-reduce;
  * model parallel (mlp.py:208-215, 247-249): activations shipped forward and
    error signals shipped back -> ``make_quantizer`` (encode -> decode round
    trip on the GPU, the single-process seam) or ``ModelParallelFC`` (the
    real sharded FC layer of BASELINE config 5).

Hook statistics (mlp.py:140-164) are accumulated on the device.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional, Union

import torch

from .codecs import DataTypeKind, DataTypeSpec, NormKind, build_codebook, decode_buffer, encode_buffer
from .errors import ConfigError

ONEBIT = "onebit"


class HookMode(str, Enum):
    NONE = "none"
    DATA_PARALLEL = "data-parallel"
    MODEL_PARALLEL = "model-parallel"


@dataclass(frozen=True)
class QuantHookConfig:
    """What gets quantised during training, and with which codec (mlp.py:97-121)."""

    mode: HookMode = HookMode.NONE
    spec: Union[DataTypeSpec, str, None] = None  # DataTypeSpec or "onebit"

    def __post_init__(self) -> None:
        object.__setattr__(self, "mode", HookMode(self.mode))
        if isinstance(self.spec, str) and self.spec != ONEBIT:
            raise ConfigError(f"string spec must be {ONEBIT!r}, got {self.spec!r}")
        if self.spec == ONEBIT and self.mode is HookMode.MODEL_PARALLEL:
            raise ConfigError("onebit quantization only supports data-parallel mode")

    @property
    def active(self) -> bool:
        return self.mode is not HookMode.NONE and self.spec is not None

    def label(self) -> str:
        if not self.active:
            return "32-bit"
        name = ONEBIT if self.spec == ONEBIT else self.spec.label()
        return f"{name} [{self.mode.value}]"


def default_hook_spec(kind: DataTypeKind, mode: HookMode) -> DataTypeSpec:
    """Normalisation defaults per codec and seam (mlp.py:399-411): tree/linear
    use absmax; exponent codecs read gradients unscaled and activations with
    a two-decade offset."""
    kind = DataTypeKind(kind)
    if kind in (DataTypeKind.DYNAMIC_TREE, DataTypeKind.LINEAR):
        return DataTypeSpec(kind, NormKind.ABSMAX)
    if HookMode(mode) is HookMode.MODEL_PARALLEL:
        return DataTypeSpec(kind, NormKind.DECADE, 2)
    return DataTypeSpec(kind, NormKind.NONE)


class HookStats:
    """Per (site, layer) sums of |x - q(x)| and |x - q(x)|/|x| over non-zero
    x (mlp.py:140-164), accumulated on the device by the a8_error_stats
    kernel; ``summary`` syncs."""

    def __init__(self) -> None:
        self._acc: dict = {}

    def _row(self, site: str, layer: int, n: int, dev: torch.device) -> torch.Tensor:
        key = (site, layer)
        if key not in self._acc:
            self._acc[key] = [torch.zeros(3, dtype=torch.float64, device=dev), 0]
        self._acc[key][1] += n
        return self._acc[key][0]

    @staticmethod
    def _flat(x: torch.Tensor) -> torch.Tensor:
        x = x.reshape(-1)
        if x.dtype not in (torch.float32, torch.float64):
            x = x.to(torch.float32)  # narrower floats widen exactly
        return x.contiguous()

    def record(self, site: str, layer: int, before: torch.Tensor, after: torch.Tensor) -> None:
        """mlp.py:146-153 with ``after`` a decoded tensor (float32 values)."""
        from .errorbench import error_sums

        b = self._flat(before)
        a = after.reshape(-1).to(device=b.device, dtype=torch.float32).contiguous()
        error_sums(b, self._row(site, layer, b.numel(), b.device), after=a, accumulate=True)

    def record_codes(self, site: str, layer: int, before: torch.Tensor, q, codebook) -> None:
        """Same sums from the 8-bit codes (decode fused into the reduction)."""
        from .errorbench import error_sums

        b = self._flat(before)
        error_sums(b, self._row(site, layer, b.numel(), b.device), codes=q.device_codes(b.device), scale=q.device_scale(b.device),
                   codebook=codebook, accumulate=True)

    def summary(self) -> dict:
        out: dict = {}
        for (site, layer) in sorted(self._acc):
            row, n = self._acc[(site, layer)]
            abs_sum, rel_sum, nnz = (float(v) for v in row.cpu())
            out.setdefault(site, []).append(
                (abs_sum / n if n else 0.0, 100.0 * rel_sum / nnz if nnz else 0.0)
            )
        return out


def make_quantizer(spec: DataTypeSpec, stats: Optional[HookStats] = None, site: str = "gradient") -> Callable:
    """GPU form of ``_make_quantizer`` (mlp.py:167-175): returns
    ``quantize(x, layer) -> decode(encode(x))`` running in the sm_100a kernels."""
    cb = build_codebook(spec)

    def quantize(x: torch.Tensor, layer: int) -> torch.Tensor:
        if x.dtype != torch.float64:  # float32 (or narrower): fused round trip when it fits
            from .codecs import _roundtrip_fused, as_device_f32

            t, shape = as_device_f32(x)
            t = t.reshape(-1)
            y = _roundtrip_fused(t, cb)
            if y is not None:
                if stats is not None:
                    stats.record(site, layer, t, y)
                return y.reshape(shape).to(x.dtype)
        q = encode_buffer(x, cb, sync=False)
        y = decode_buffer(q, cb)
        if stats is not None:
            stats.record_codes(site, layer, q._keepalive, q, cb)
        q._finish()  # InputError for NaN/Inf, as encode_buffer raises in mlp.py:171
        return y.to(x.dtype)

    return quantize


class ModelParallelFC:
    """Column-sharded fully connected layer with 8-bit activations on the
    wire (BASELINE config 5; the model-parallel seam of mlp.py:208-215 and
    247-249, where the reference round-trips the tensors that cross devices).

    Rank r of N owns ``weight_shard`` = W[:, r*k:(r+1)*k] (in x out_shard).
      forward(x)   y_r = x @ W_r; the shards are 8-bit all-gathered (one
                   absmax scale per shard) and concatenated: y = [q(y_0) .. q(y_N-1)]
      backward(dy) dx_r = dy[:, shard r] @ W_r^T is a partial of dx; the
                   partials are summed through the compressed exchange
                   (op="sum"): dx = sum_r q(dx_r), rank order, float32;
                   dW_r = x^T dy_r stays local.
    ``comm`` is the collective backend (torch.distributed by default).
    ``activation="relu"``: the shipped tensor is the hidden activation
    h_r = np.maximum(y_r, 0) [* mask_r] (mlp.py:205-209), produced by
    ``relu_absmax`` so that its max comes with it and the encode is one pass
    (absmax specs); backward then takes dy w.r.t. h.
    """

    def __init__(self, weight_shard: torch.Tensor, spec: DataTypeSpec, group=None, comm=None, codec=None,
                 activation: Optional[str] = None):
        from .exchange import CompressedAllGather, GradientExchange

        if activation not in (None, "relu"):
            raise ConfigError(f"activation must be None or 'relu', got {activation!r}")
        self.w = weight_shard
        self.spec = spec
        self.activation = activation
        self.gather = CompressedAllGather(spec, group, codec=codec, comm=comm)
        self.reduce = GradientExchange(spec, group, mode="allgather", op="sum", check="sync", codec=codec, comm=comm)
        self._x = None
        self._gate = None

    def forward(self, x: torch.Tensor, mask: Optional[torch.Tensor] = None) -> torch.Tensor:
        """``mask``: this rank's dropout multipliers (same shape as y_r), relu only."""
        from .produce import relu_absmax

        self._x = x
        y_r = (x @ self.w).contiguous()
        if self.activation is None:
            if mask is not None:
                raise ConfigError("mask needs activation='relu'")
            parts = self.gather(y_r)
        else:
            gate = (y_r > 0).to(torch.float32)  # d h / d y = mask * (y > 0) (mlp.py:250-253)
            self._gate = gate if mask is None else gate * mask
            h_r, amax = relu_absmax(y_r, mask, out=y_r)
            parts = self.gather(h_r, amax=amax if self.spec.normalization is NormKind.ABSMAX else None)
        return torch.cat(parts, dim=1)

    def backward(self, dy: torch.Tensor):
        n_r = self.w.shape[1]
        nranks, rank = self.gather.comm.world()
        dy_r = dy[:, rank * n_r:(rank + 1) * n_r]
        if self._gate is not None:
            dy_r = dy_r * self._gate
        dw = self._x.t() @ dy_r
        dx = (dy_r @ self.w.t()).contiguous()
        self.reduce([dx])
        return dx, dw
