"""Host cost of one GradientExchange call at N > 1 (AlexNet shapes) with a
no-op collective stand-in (world N, rank 0): the time Python + the C
launchers take to enqueue the step's encode, K all-gathers and K decodes
(allgather) or the two rounds (two_round), against its GPU time."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import paper_1511_04561_b200 as A  # noqa: E402
from prof_codec import ALEXNET  # noqa: E402


class NoopComm:
    def __init__(self, n):
        self.n = n

    def world(self):
        return self.n, 0

    class _H:
        def wait(self):
            pass

    def all_gather(self, out, slot):
        pass

    def all_gather_async(self, out, slot):
        return self._H()

    def all_to_all(self, recv, send):
        pass


def main():
    dev = torch.device("cuda", 0)
    gs = [torch.randn(s, device=dev) * 1e-3 for s in ALEXNET]
    outs = [torch.empty_like(g) for g in gs]
    res = []
    for n, mode in ((2, "allgather"), (8, "allgather"), (4, "two_round"), (8, "two_round")):
        ex = A.GradientExchange(A.parse_spec("dynamic-tree/absmax"), mode=mode, check="deferred", comm=NoopComm(n))
        for _ in range(5):
            ex(gs, out=outs)
        torch.cuda.synchronize()
        torch.cuda._sleep(int(2e9 * 0.1))  # a busy GPU: the host enqueues without back-pressure
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
        ex.synchronize()
        res.append({"n": n, "mode": mode, "host_enqueue_us_per_step": round(host_us, 1),
                    "gpu_us_per_step_no_comm": round(e0.elapsed_time(e1) / 20 * 1e3, 1)})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
