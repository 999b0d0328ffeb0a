"""Host-side cost of one GradientExchange call (AlexNet shapes, N=1): the
time Python + the C launcher take to enqueue a step, against the GPU time of
the step.  If the host is slower than the GPU, the step is host-bound."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1511_04561_b200 as A  # noqa: E402
from prof_codec import ALEXNET  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    gs = [torch.randn(s, device=dev) * 1e-3 for s in ALEXNET]
    outs = [torch.empty_like(g) for g in gs]
    kw = {}
    if "--graph" in sys.argv:
        kw["graph"] = True
    ex = A.GradientExchange(A.parse_spec("dynamic-tree/absmax"), check="deferred", **kw)
    for _ in range(5):
        ex(gs, out=outs)
    torch.cuda.synchronize()
    # a long GPU-side delay so the host enqueues against a busy GPU
    torch.cuda._sleep(int(2e9 * 0.05))
    t0 = time.perf_counter()
    for _ in range(20):
        ex(gs, out=outs)
    host_us = (time.perf_counter() - t0) / 20 * 1e6
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e9 * 0.01))
    e0.record()
    for _ in range(20):
        ex(gs, out=outs)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"graph": bool(kw), "host_enqueue_us_per_step": host_us,
                      "gpu_us_per_step_busy_queue": e0.elapsed_time(e1) / 20 * 1e3}))


if __name__ == "__main__":
    main()
