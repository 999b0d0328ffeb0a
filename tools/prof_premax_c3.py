"""Config-3 one-pass (premax) encode and two-pass encode, graph-replayed after a
256 MB L2 flush, mean of 40 (bench.py codec_sweep.premax.c3 takes the median of 15):
    python tools/prof_premax_c3.py      (env knobs: A8_PREMAX_HOLD, A8_PREMAX_TABLES)"""
import json, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan  # noqa
dev = torch.device("cuda", 0)
import os  # noqa
FLUSH_READ = os.environ.get("FLUSH", "read") == "read"  # FLUSH=write: the old written flush
flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
sink = torch.zeros((), dtype=torch.float32, device=dev)


def time_graph(fn, reps=40):
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
        if FLUSH_READ:
            torch.sum(flush, 0, out=sink)
        else:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts))  # mean: the event clock ticks in ~2 us steps


spec = A.parse_spec("dynamic-tree/absmax")
ts = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in bench.ALEXNET]
plan = make_plan(tuple(t.numel() for t in ts), 1)
C, P = plan.flat, plan.allgather_block()
slab = torch.zeros(P, dtype=torch.uint8, device=dev)
cb, codec, idx = A.build_codebook(spec), CudaSegmentCodec(), list(range(plan.nseg))
m = A.scale_absmax_(ts, 1.0)


def enc(**kw):
    codec.encode(ts, plan.offs, idx, cb, slab, 0, C, C, C, 0, 1, C + 4 * plan.status_slot, **kw)


print(json.dumps({"premax_us": round(time_graph(lambda: enc(amax=m)) * 1e3, 1),
                  "two_pass_us": round(time_graph(enc) * 1e3, 1)}))
