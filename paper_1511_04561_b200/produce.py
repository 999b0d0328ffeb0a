"""Producer passes that emit the per-tensor max |y| as they write y, so the
8-bit encode that follows is one pass (a8_produce_absmax + a8_encode_premax,
SURVEY 8(f) row 4).

The reference encodes with scale = max|x| (codecs.py:237-241), which costs
an extra read of x before the encode when x is larger than L2.  When the
kernel that writes x already streams every element, the max comes free:

  * ``scale_absmax_(grads, alpha)``: the data-parallel gradient pre-scaling
    (1/N averaging, loss-scale removal) in place, with the maxima;
    ``alpha=1`` is the max pass alone (no stores);
  * ``relu_absmax(z, mask)``: the model-parallel forward producer,
    ``h = np.maximum(z, 0) * mask`` (mlp.py:205-207), whose output is the
    activation the forward hook ships (mlp.py:208-209).

The maxima come back as a float32 tensor for ``GradientExchange(...)(...,
amax=)``, ``CompressedAllGather(...)(..., amax=)`` and ``encode_buffer(...,
amax=)``.  No CPU path: CUDA tensors only.
"""

from __future__ import annotations

from typing import Optional, Sequence, Tuple

import torch

from . import _native as N
from .errors import UsageError


def _check(ts, what: str):
    dev = ts[0].device
    for t in ts:
        if t.dtype != torch.float32 or not t.is_contiguous() or t.device != dev or dev.type != "cuda":
            raise UsageError(f"{what} needs contiguous float32 CUDA tensors on one device")
    return dev


def _launch(xs, ys, masks, op: int, alpha: float) -> torch.Tensor:
    dev = xs[0].device
    out = torch.empty(len(xs), dtype=torch.int32, device=dev)
    segs = (N.ProdSeg * len(xs))()
    for i, (x, y) in enumerate(zip(xs, ys)):
        segs[i] = N.ProdSeg(x.data_ptr(), y.data_ptr(), 0 if masks is None else masks[i].data_ptr(), x.numel())
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(N.lib.a8_produce_absmax(segs, len(xs), op, float(alpha), out.data_ptr(), stream))
    return out.view(torch.float32)


def scale_absmax_(tensors: Sequence[torch.Tensor], alpha: float = 1.0) -> torch.Tensor:
    """t *= alpha (float32, round to nearest) for every tensor, in place; returns
    float32 [len(tensors)] with max|t| of each result (NaN if it holds NaN)."""
    ts = list(tensors)
    if not ts:
        raise UsageError("scale_absmax_ needs at least one tensor")
    _check(ts, "scale_absmax_")
    return _launch(ts, ts, None, N.A8_PRODUCE_SCALE, alpha)


def relu_absmax(z: torch.Tensor, mask: Optional[torch.Tensor] = None,
                out: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """h = np.maximum(z, 0) [* mask] (mlp.py:205-207) in float32, and max|h|
    as a float32 [1] tensor.  ``out`` may be ``z`` (in place)."""
    _check([z] + ([mask] if mask is not None else []) + ([out] if out is not None else []), "relu_absmax")
    if mask is not None and mask.numel() != z.numel():
        raise UsageError("mask must have as many elements as z")
    h = torch.empty_like(z) if out is None else out
    if h.numel() != z.numel():
        raise UsageError("out must have as many elements as z")
    op = N.A8_PRODUCE_RELU if mask is None else N.A8_PRODUCE_RELU_MASK
    return h, _launch([z], [h], None if mask is None else [mask], op, 1.0)
