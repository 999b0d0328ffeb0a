"""BASELINE config 4: codec bandwidth sweep, n = 2^10 .. 2^30, four kinds.

    python tools/sweep_config4.py [--reps 7] [--max-log2 30] > profiles/<tag>_sweep_config4.jsonl

Kernel time without host overhead: each encode and decode is captured in a
CUDA graph between external CUDA events on the launching stream; every rep
first flushes L2 (writes a 256 MB buffer, outside the events), then replays
the graph once and reads the event times.  GB/s at algorithmic bytes: encode
4n + n (+4 per scale), decode n + 4n.  Inputs N(0,1) with seed k (SURVEY
8(d) C4).
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
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan  # noqa: E402

SPECS = ["dynamic-tree/absmax", "linear/absmax", "static-tree/decade+1", "mantissa/decade+1"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--max-log2", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    codec = CudaSegmentCodec()
    for k in range(10, a.max_log2 + 1, 2):
        n = 1 << k
        gen = torch.Generator(device=dev).manual_seed(k)
        x = torch.randn(n, device=dev, generator=gen)
        out = torch.empty_like(x)
        plan = make_plan([n], 1)
        B = plan.allgather_block()
        buf = torch.zeros(B, dtype=torch.uint8, device=dev)
        st = torch.zeros(1, dtype=torch.int32, device=dev)
        for label in SPECS:
            cb = A.build_codebook(A.parse_spec(label))
            s = torch.cuda.Stream(dev)
            ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]

            def step():
                ev[0].record()
                codec.encode([x], plan.offs, [0], cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, 1,
                             plan.flat + 4 * plan.status_slot)
                ev[1].record()
                codec.decode([out], plan.offs, [0], cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, B, 1, 1,
                             plan.status_slot, 1, st)
                ev[2].record()

            with torch.cuda.stream(s):  # eager warm-up on the capture stream (workspace, tables)
                step()
                step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                step()
            enc, dec = [], []
            for _ in range(a.reps):
                flush.fill_(1)
                g.replay()
                torch.cuda.synchronize()
                enc.append(ev[0].elapsed_time(ev[1]))
                dec.append(ev[1].elapsed_time(ev[2]))
            e_ms, d_ms = float(np.median(enc)), float(np.median(dec))
            print(json.dumps({"n": n, "log2": k, "spec": label, "encode_us": e_ms * 1e3, "decode_us": d_ms * 1e3,
                              "encode_GBps": (5.0 * n + 4) / (e_ms * 1e-3) / 1e9,
                              "decode_GBps": 5.0 * n / (d_ms * 1e-3) / 1e9,
                              "roundtrip_GBps": 10.0 * n / ((e_ms + d_ms) * 1e-3) / 1e9,
                              "l2": "flushed before every rep"}), flush=True)
        del x, out, buf


if __name__ == "__main__":
    main()
