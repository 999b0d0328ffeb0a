"""Golden vectors for the GPU error bench, from the REAL reference.

Run in the build container only (``/root/reference`` is absent on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_errorbench.py

Writes ``tests/golden/errorbench.json``:
  suite_seed0      run_error_suite(seed=0, count=1e6) reports, reports_to_csv
                   and format_table text (errorbench.py:142-206)
  suite_seed5      run_error_suite(seed=5, count=20_000) (test_errorbench.py:146-152)
  cells            measure_error on seeded inputs (errorbench.py:79-99): the
                   naive-rescan input of test_errorbench.py:63-66, float64
                   input, zeros mixed in, single elements, power-of-two scales
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("APPROX8_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from approx8 import errorbench as EB  # noqa: E402
from approx8.codecs import DataTypeKind, DataTypeSpec, NormKind  # noqa: E402

OUT = Path(__file__).resolve().parent / "errorbench.json"


def rep(r):
    return {"dist": r.sample_label, "spec": r.spec.label(), "n": r.count, "seed": r.seed,
            "mean_abs_error": r.mean_abs_error, "mean_rel_error_pct": r.mean_rel_error_pct}


def cell_inputs():
    """(name, array) pairs; regenerated identically by tests/test_gpu_errorbench.py."""
    rng = np.random.default_rng(11)
    yield "rescan_normal1000", rng.normal(size=1000).astype(np.float32)
    rng = np.random.default_rng(12)
    yield "normal4096_x1024", (rng.normal(size=4096).astype(np.float32) * np.float32(1024.0))
    rng = np.random.default_rng(13)
    x = rng.normal(0, 0.01, size=100_003)
    x[::7] = 0.0
    yield "f64_zeros", x  # float64 input, 1/7 zeros
    yield "single", np.array([0.3], dtype=np.float32)
    yield "allzero", np.zeros(257, dtype=np.float32)
    rng = np.random.default_rng(14)
    yield "uniform_1e6", rng.random(1_000_000).astype(np.float32)


SPECS = [("dynamic-tree", "absmax", 0), ("linear", "absmax", 0), ("mantissa", "decade", 1),
         ("static-tree", "decade", 1), ("dynamic-tree", "none", 0), ("mantissa", "none", 0)]


def main():
    out = {}
    reps = EB.run_error_suite(seed=0, count=1_000_000)
    out["suite_seed0"] = {"reports": [rep(r) for r in reps], "csv": EB.reports_to_csv(reps),
                          "table": EB.format_table(reps)}
    reps = EB.run_error_suite(seed=5, count=20_000)
    out["suite_seed5"] = {"reports": [rep(r) for r in reps], "csv": EB.reports_to_csv(reps)}
    cells = []
    for name, x in cell_inputs():
        for kind, norm, dec in SPECS:
            spec = DataTypeSpec(DataTypeKind(kind), NormKind(norm), dec)
            r = EB.measure_error(x, spec)
            cells.append({"input": name, "spec": spec.label(), "mean_abs_error": r.mean_abs_error,
                          "mean_rel_error_pct": r.mean_rel_error_pct, "count": r.count})
    out["cells"] = cells
    OUT.write_text(json.dumps(out, indent=1) + "\n")
    print(f"wrote {OUT} ({len(cells)} cells)")


if __name__ == "__main__":
    main()
