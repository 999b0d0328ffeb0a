"""K5 decode-reduce (the exchange's fused decode + rank-ordered sum + 1/N):
one GPU, N code slabs in one buffer (as after the all-gather), AlexNet shapes.
Graph-captured kernel events, L2 flushed before each rep.  Algorithmic bytes
(SURVEY 8(d)): N*n codes read + 4n written (+ scales)."""
import json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan  # noqa
from prof_codec import ALEXNET  # noqa

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
spec = A.parse_spec("dynamic-tree/absmax")
cb = A.build_codebook(spec)
codec = CudaSegmentCodec()
xs = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in ALEXNET]
outs = [torch.empty_like(x) for x in xs]
n = sum(x.numel() for x in xs)
for N in (1, 2, 4, 8):
    plan = make_plan([x.numel() for x in xs], N)
    P = plan.allgather_block()
    buf = torch.zeros(N * P, dtype=torch.uint8, device=dev)
    idx = list(range(len(xs)))
    for r in range(N):  # every rank's slab (same data: the kernel work is identical)
        codec.encode(xs, plan.offs, idx, cb, buf, r * P, r * P + plan.flat, plan.flat, plan.flat, 0, 1,
                     r * P + plan.flat + 4 * plan.status_slot)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream(dev)
    ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(2)]

    def step():
        ev[0].record()
        codec.decode(outs, plan.offs, idx, cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, P, N, 1,
                     plan.status_slot, 1, st)
        ev[1].record()

    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    ts = []
    for _ in range(7):
        flush.fill_(1)
        g.replay()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ms = float(np.median(ts))
    alg = (N + 4.0) * n
    print(json.dumps({"nranks": N, "n": n, "decode_reduce_us": ms * 1e3, "alg_bytes": alg,
                      "GBps": alg / (ms * 1e-3) / 1e9}), flush=True)
