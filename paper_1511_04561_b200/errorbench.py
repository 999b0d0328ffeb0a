"""GPU error bench: round-trip error aggregates of the 8-bit codecs
(reference: approx8/errorbench.py).

Same names, arguments, validation and report formats as the reference
module.  The samples are drawn on the host with the reference's own
generator (NumPy ``default_rng``, errorbench.py:59-66) so every cell sees
the same bytes; the round trip and the error sums run on the GPU:

  encode (a8_encode / a8_encode_f64)  ->  a8_error_stats (fused decode +
  |x - d| and |x - d|/|x| float64 sums, nothing written back but 3 doubles)

The per-element arithmetic is the reference's; the sums are a fixed-order
tree rather than NumPy's pairwise sum, so aggregates agree to float64
rounding (the reference's own tests compare at rel 1e-12).
"""

from __future__ import annotations

import csv
import io
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np
import torch

from . import _native as N
from .codecs import DataTypeKind, DataTypeSpec, NormKind, _cuda_device, _stream, build_codebook, encode_buffer
from .errors import ConfigError, UsageError

DIST_UNIFORM01 = "uniform01"
DIST_NORMAL = "normal"


@dataclass(frozen=True)
class SampleSpec:
    """A reproducible draw: distribution, size, and seed (errorbench.py:34-56)."""

    distribution: str
    count: int
    seed: int
    mean: float = 0.0
    sigma: float = 1.0

    def __post_init__(self) -> None:
        if self.distribution not in (DIST_UNIFORM01, DIST_NORMAL):
            raise ConfigError(f"unknown distribution {self.distribution!r}")
        if self.count < 1:
            raise ConfigError(f"sample count must be >= 1, got {self.count}")
        if self.sigma <= 0:
            raise ConfigError(f"sigma must be > 0, got {self.sigma}")

    def label(self) -> str:
        if self.distribution == DIST_UNIFORM01:
            return "U(0,1)"
        return f"N({self.mean:g},{self.sigma:g}^2)"


def sample(spec: SampleSpec) -> np.ndarray:
    """The sample as float32, deterministically from ``spec.seed``
    (errorbench.py:59-66: float64 draws from ``default_rng``, cast to float32)."""
    rng = np.random.default_rng(spec.seed)
    if spec.distribution == DIST_UNIFORM01:
        data = rng.random(spec.count, dtype=np.float64)
    else:
        data = rng.normal(spec.mean, spec.sigma, spec.count)
    return data.astype(np.float32)


@dataclass(frozen=True)
class ErrorReport:
    spec: DataTypeSpec
    mean_abs_error: float
    mean_rel_error_pct: float
    count: int
    sample_label: str = ""
    seed: int = 0


_ws_lock = threading.Lock()
_ws_cache: dict = {}


def error_workspace(dev: torch.device, stream: int) -> torch.Tensor:
    """Zero-filled scratch of a8_error_stats for (device, stream); the kernel
    leaves it zeroed."""
    key = (dev.index, stream)
    with _ws_lock:
        ws = _ws_cache.get(key)
        if ws is None:
            ws = torch.zeros(int(N.lib.a8_error_workspace_bytes()), dtype=torch.uint8, device=dev)
            _ws_cache[key] = ws
    return ws


def error_sums(x: torch.Tensor, out: torch.Tensor, *, codes=None, scale=None, codebook=None, after=None,
               accumulate: bool = False) -> None:
    """Launch a8_error_stats on ``x`` (a contiguous float32/float64 CUDA
    tensor) against either 8-bit ``codes`` + device ``scale`` (fused decode)
    or a decoded float32 tensor ``after``.  ``out`` (float64[3], same device)
    receives or accumulates [sum |x-d|, sum |x-d|/|x| over x != 0, #(x != 0)]."""
    dev = x.device
    if x.dtype not in (torch.float32, torch.float64) or not x.is_contiguous():
        raise UsageError("error_sums: x must be a contiguous float32 or float64 CUDA tensor")
    if out.dtype != torch.float64 or out.numel() != 3 or out.device != dev:
        raise UsageError("error_sums: out must be float64[3] on x's device")
    n = x.numel()
    with torch.cuda.device(dev):
        stream = _stream(dev)
        ws = error_workspace(dev, stream)
        if codes is not None:
            book, _ = codebook.device_tables(dev)
            args = (codes.data_ptr(), scale.data_ptr(), book.data_ptr(), None)
        else:
            if after.dtype != torch.float32 or not after.is_contiguous() or after.numel() != n:
                raise UsageError("error_sums: after must be a contiguous float32 tensor of x's size")
            args = (None, None, None, after.data_ptr())
        N.check(N.lib.a8_error_stats(x.data_ptr(), int(x.dtype == torch.float64), n, *args, out.data_ptr(),
                                     int(accumulate), ws.data_ptr(), ws.numel(), stream))


def measure_error(x, spec: DataTypeSpec, *, device=None) -> ErrorReport:
    """Round-trip ``x`` through the codec on the GPU and report the error
    aggregates (errorbench.py:79-99): mean |x - q(x)| over every element and
    the mean of |x - q(x)|/|x| in percent over the non-zero elements."""
    count = x.numel() if isinstance(x, torch.Tensor) else int(np.asarray(x).size)
    if count == 0:
        raise UsageError("cannot measure error of an empty buffer")
    cb = build_codebook(spec)
    q = encode_buffer(x, cb, device=device, sync=False)
    xd = q._keepalive  # the flat device input the encoder read (float32, or float64 input as is)
    dev = xd.device
    out = torch.empty(3, dtype=torch.float64, device=dev)
    error_sums(xd, out, codes=q.codes_device, scale=q.scale_tensor, codebook=cb)
    q._finish()  # non-finite input -> InputError, as roundtrip raises in the reference
    abs_sum, rel_sum, nnz = (float(v) for v in out.cpu())
    rel_pct = float(rel_sum / nnz * 100.0) if nnz else 0.0
    return ErrorReport(spec=spec, mean_abs_error=abs_sum / count, mean_rel_error_pct=rel_pct, count=count)


# Suite layout: distributions x codecs, in the order results are reported
# (errorbench.py:102-115).
SUITE_DISTRIBUTIONS: tuple[tuple[str, dict], ...] = (
    (DIST_UNIFORM01, {}),
    (DIST_NORMAL, {"mean": 0.0, "sigma": 1.0}),
    (DIST_NORMAL, {"mean": 0.0, "sigma": 10.0}),
    (DIST_NORMAL, {"mean": 0.0, "sigma": 0.2}),
)

SUITE_KINDS: tuple[DataTypeKind, ...] = (
    DataTypeKind.DYNAMIC_TREE,
    DataTypeKind.LINEAR,
    DataTypeKind.MANTISSA,
    DataTypeKind.STATIC_TREE,
)


def suite_spec(kind: DataTypeKind, dist: str, params: dict) -> DataTypeSpec:
    """The normalisation each codec wears in the grid (errorbench.py:117-127):
    absmax for tree/linear, one decade for the exponent codecs (two for the
    sigma-10 normal)."""
    kind = DataTypeKind(kind)
    if kind in (DataTypeKind.DYNAMIC_TREE, DataTypeKind.LINEAR):
        return DataTypeSpec(kind, NormKind.ABSMAX)
    decades = 2 if params.get("sigma", 1.0) >= 10.0 else 1
    return DataTypeSpec(kind, NormKind.DECADE, decades)


def worker_count(n_tasks: int) -> int:
    """Host thread-pool width for sampling, capped by APPROX8_THREADS
    (errorbench.py:130-139)."""
    cap = os.environ.get("APPROX8_THREADS")
    limit = os.cpu_count() or 1
    if cap is not None:
        try:
            limit = max(1, int(cap))
        except ValueError as exc:
            raise ConfigError(f"APPROX8_THREADS must be an integer, got {cap!r}") from exc
    return max(1, min(limit, n_tasks))


def run_error_suite(seed: int = 0, count: int = 1_000_000, kinds: Sequence[DataTypeKind] = SUITE_KINDS,
                    *, device=None) -> list[ErrorReport]:
    """The distribution-by-codec grid (errorbench.py:142-171).  Cell i draws
    from ``seed + i``; samples are drawn on a host thread pool, each cell is
    measured on the GPU as soon as its sample is ready, in cell order."""
    cells = []
    for d_idx, (dist, params) in enumerate(SUITE_DISTRIBUTIONS):
        for k_idx, kind in enumerate(kinds):
            cell_seed = seed + d_idx * len(kinds) + k_idx
            sspec = SampleSpec(dist, count, cell_seed, **params)
            cells.append((sspec, suite_spec(kind, dist, params)))
    dev = _cuda_device(device)
    out = []
    with ThreadPoolExecutor(max_workers=worker_count(len(cells))) as pool:
        samples = [pool.submit(sample, sspec) for sspec, _ in cells]
        for (sspec, dspec), fut in zip(cells, samples):
            r = measure_error(torch.from_numpy(fut.result()).to(dev), dspec)
            out.append(ErrorReport(spec=r.spec, mean_abs_error=r.mean_abs_error,
                                   mean_rel_error_pct=r.mean_rel_error_pct, count=r.count,
                                   sample_label=sspec.label(), seed=sspec.seed))
    return out


CSV_HEADER = ("distribution", "datatype", "n", "mean_abs_error", "mean_rel_error_pct", "seed")


def reports_to_csv(reports: Iterable[ErrorReport]) -> str:
    """CSV rendering, byte-compatible with errorbench.py:177-192."""
    buf = io.StringIO()
    writer = csv.writer(buf, lineterminator="\n")
    writer.writerow(CSV_HEADER)
    for r in reports:
        writer.writerow((r.sample_label, r.spec.label(), r.count, f"{r.mean_abs_error:.6e}",
                         f"{r.mean_rel_error_pct:.4f}", r.seed))
    return buf.getvalue()


def format_table(reports: Sequence[ErrorReport]) -> str:
    """Aligned text rendering grouped by distribution (errorbench.py:195-206)."""
    lines = [f"{'distribution':<14}{'datatype':<24}{'mean abs err':>14}{'mean rel err %':>16}"]
    for r in reports:
        lines.append(f"{r.sample_label:<14}{r.spec.label():<24}"
                     f"{r.mean_abs_error:>14.3e}{r.mean_rel_error_pct:>16.3f}")
    return "\n".join(lines) + "\n"


def main(argv=None) -> int:
    """``python -m paper_1511_04561_b200.errorbench`` -- the reference CLI's
    ``bench-error`` (cli.py:119-125, 248-253) on the GPU."""
    import argparse

    ap = argparse.ArgumentParser(prog="paper_1511_04561_b200.errorbench",
                                 description="distribution x codec error grid (GPU)")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--table", action="store_true", help="aligned text instead of CSV")
    ap.add_argument("--out")
    a = ap.parse_args(argv)
    reports = run_error_suite(seed=a.seed, count=a.n)
    text = format_table(reports) if a.table else reports_to_csv(reports)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text, end="")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
