"""The codec_sweep's per-block cases alone (bench.py method: one public-API
call per case, CUDA-graph replayed between events, 256 MB L2 flush before
each replay, median of 7)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def time_graph(fn, reps=7):
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
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
for k in (28, 30):
    x = torch.randn(1 << k, device=dev)
    y = torch.empty_like(x)
    for b in (4096, 1024):
        box = {}
        te = time_graph(lambda: box.__setitem__("q", A.encode_buffer(x, cb, sync=False, block_size=b)))
        box["q"]._finish()
        td = time_graph(lambda: A.decode_buffer(box["q"], cb, out=y))
        print(json.dumps({"n": 1 << k, "block": b, "encode_us": te * 1e3, "decode_us": td * 1e3}))
        del box
