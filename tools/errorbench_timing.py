"""Time the GPU error bench (one GPU).

    python tools/errorbench_timing.py [--n 25000000]

Per suite cell: the sample is drawn on the host (not timed) and copied to the
device; the timed region is measure_error's device work (encode + fused
error sums, CUDA events, median of 5) on the resident input.  Prints JSON
lines and the table.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1511_04561_b200 as A  # noqa: E402
from paper_1511_04561_b200 import errorbench as EB  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=25_000_000)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    cells = []
    for d_idx, (dist, params) in enumerate(EB.SUITE_DISTRIBUTIONS):
        for k_idx, kind in enumerate(EB.SUITE_KINDS):
            cells.append((EB.SampleSpec(dist, a.n, d_idx * 4 + k_idx, **params), EB.suite_spec(kind, dist, params)))
    tot = 0.0
    reports = []
    for sspec, dspec in cells:
        x = torch.from_numpy(EB.sample(sspec)).to(dev)
        for _ in range(2):
            r = EB.measure_error(x, dspec)
        ms = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = EB.measure_error(x, dspec)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        m = float(np.median(ms))
        tot += m
        absmax = dspec.normalization == A.NormKind.ABSMAX
        nbytes = a.n * ((9 if absmax else 5) + 5)  # encode (max pass + encode) + stats (x + codes)
        reports.append(EB.ErrorReport(r.spec, r.mean_abs_error, r.mean_rel_error_pct, r.count, sspec.label(), sspec.seed))
        print(json.dumps({"cell": f"{sspec.label()} {dspec.label()}", "n": a.n, "gpu_ms": m,
                          "GBps_algorithmic": nbytes / (m * 1e-3) / 1e9,
                          "mean_abs_error": r.mean_abs_error, "mean_rel_error_pct": r.mean_rel_error_pct}), flush=True)
    print(json.dumps({"suite_gpu_ms": tot, "n": a.n, "cells": len(cells)}), flush=True)
    sys.stdout.write(EB.format_table(reports))


if __name__ == "__main__":
    main()
