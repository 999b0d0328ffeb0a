"""Per-block decode time at 2^28 / 2^30 for B = 1024 / 2048 / 4096 (graph-replayed, L2 flushed)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cb = A.build_codebook(A.parse_spec("dynamic-tree/absmax"))


def tg(fn, reps=7):
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream(dev).wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for k in (28, 30):
    x = torch.randn(1 << k, device=dev)
    y = torch.empty_like(x)
    for b in (1024, 2048, 4096):
        q = A.encode_buffer(x, cb, block_size=b)
        print(k, b, "decode us", round(tg(lambda: A.decode_buffer(q, cb, out=y)), 1), flush=True)
    del x, y
