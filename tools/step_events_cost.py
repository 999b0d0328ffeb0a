"""Bench-step cost of the per-kernel timing events captured in the graph:
the C3 N=1 exchange graph with and without the event nodes (one B200)."""
import faulthandler
import sys
from pathlib import Path

faulthandler.enable()

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1511_04561_b200 as A  # noqa: E402

dev = torch.device("cuda", 0)
host = bench.alexnet_grads(0)
grads = [torch.from_numpy(g).to(dev) for g in host]
outs = [torch.empty_like(g) for g in grads]
spec = A.parse_spec("dynamic-tree/absmax")


def timed(ex, steps=50):
    for _ in range(5):
        ex(grads, out=outs)
    ex.synchronize()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        ex(grads, out=outs)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


class Evented:
    """The bench's TimedCodec: the events must outlive the graph capture."""

    def __init__(self, codec):
        self.c = codec
        self.keep = []

    def _ev(self, fn, *a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
        e0.record(); fn(*a, **k); e1.record()
        self.keep.append((e0, e1))

    def encode(self, *a, **k):
        self._ev(self.c.encode, *a, **k)

    def decode(self, *a, **k):
        self._ev(self.c.decode, *a, **k)


for rep in range(3):
    print("rep", rep, flush=True)
    ex = A.GradientExchange(spec, graph=True, check="deferred")
    plain = timed(ex)
    print("plain", plain, flush=True)
    ex2 = A.GradientExchange(spec, graph=True, check="deferred")
    ex2.codec = Evented(ex2.codec)
    ev = timed(ex2)
    print("evented", ev, flush=True)
    ex3 = A.GradientExchange(spec, graph=True, check="none")
    nochk = timed(ex3)
    print(f"graph step: no events {plain:.1f} us, 4 event nodes {ev:.1f} us, check=none {nochk:.1f} us")
