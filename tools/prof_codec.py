"""Codec micro-benchmark / profiling driver (one GPU).

    python tools/prof_codec.py --case alexnet|single|static|sweep [--iters N]

Times a8_encode / a8_decode launches with CUDA events and prints GB/s at
algorithmic bytes (encode 5 B/elem, decode 5 B/elem).  Used under ncu to
capture the kernels (short --iters).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1511_04561_b200 as A  # noqa: E402
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan  # noqa: E402

ALEXNET = [(64, 3, 11, 11), (64,), (192, 64, 5, 5), (192,), (384, 192, 3, 3), (384,),
           (256, 384, 3, 3), (256,), (256, 256, 3, 3), (256,), (4096, 9216), (4096,),
           (4096, 4096), (4096,), (1000, 4096), (1000,)]


def run(sizes, spec, iters, dev):
    gen = torch.Generator(device=dev).manual_seed(0)
    xs = [torch.randn(int(np.prod(s)), device=dev, generator=gen) * 1e-3 for s in sizes]
    outs = [torch.empty_like(x) for x in xs]
    plan = make_plan([x.numel() for x in xs], 1)
    cb = A.build_codebook(spec)
    codec = CudaSegmentCodec()
    B = plan.allgather_block()
    buf = torch.zeros(B, dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    idx = list(range(len(xs)))
    n = sum(x.numel() for x in xs)

    kw = {"amax": A.scale_absmax_(xs, 1.0)} if PREMAX else {}

    def enc():
        codec.encode(xs, plan.offs, idx, cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, 1,
                     plan.flat + 4 * plan.status_slot, **kw)

    def dec():
        codec.decode(outs, plan.offs, idx, cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, B, 1, 1,
                     plan.status_slot, 1, st)

    for _ in range(3):
        enc()
        dec()
    torch.cuda.synchronize()
    res = {}
    for name, fn in (("encode", enc), ("decode", dec)):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
        for e0, e1 in evs:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in evs]))
        res[name] = {"ms": ms, "GBps": 5.0 * n / (ms * 1e-3) / 1e9}
    if TRACE:
        import ctypes as C

        from paper_1511_04561_b200 import _native as N
        from paper_1511_04561_b200.codecs import workspace

        enc()
        torch.cuda.synchronize()
        ws = workspace(dev, torch.cuda.current_stream(dev).cuda_stream, len(xs))
        out = (C.c_uint64 * (4 + 4 * len(xs)))()
        N.check(N.lib.a8_encode_trace(ws.data_ptr(), len(xs), out))
        t0 = out[0]
        order = sorted(range(len(xs)), key=lambda i: xs[i].numel())
        res["trace"] = {
            "kernel_us": (out[1] - t0) / 1e3, "wait_cta_us": out[2] / 1e3, "waits": out[3],
            "builds": [{"n": xs[order[k]].numel(), "start_us": round((out[4 + 4 * k] - t0) / 1e3, 2),
                        "thr_us": round((out[5 + 4 * k] - out[4 + 4 * k]) / 1e3, 2),
                        "fill_us": round((out[6 + 4 * k] - out[5 + 4 * k]) / 1e3, 2),
                        "pub_us": round((out[7 + 4 * k] - out[6 + 4 * k]) / 1e3, 2)}
                       for k in range(len(xs)) if out[4 + 4 * k] >= t0],
        }
    return n, res


TRACE = "--trace" in sys.argv
PREMAX = "--premax" in sys.argv or os.environ.get("A8_PREMAX") == "1"  # supplied maxima (a8_encode_premax)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="alexnet")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--spec", default="dynamic-tree/absmax")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--premax", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    spec = A.parse_spec(a.spec)
    if a.case == "alexnet":
        cases = [("alexnet", ALEXNET)]
    elif a.case == "mlpcodec":
        cases = [("mlp", [(784, 1200), (1200,), (1200, 1200), (1200,), (1200, 10), (10,)])]
    elif a.case == "small":
        cases = [("2^16", [(1 << 16,)]), ("c1_2^20", [(1 << 20,)]), ("2^22", [(1 << 22,)])]
    elif a.case == "single":
        cases = [("single_2^26", [(1 << 26,)])]
    elif a.case == "big":
        cases = [("single_2^26", [(1 << 26,)]), ("single_2^28", [(1 << 28,)]), ("single_2^30", [(1 << 30,)])]
    elif a.case == "bw":
        # torch reference kernels on 2^28 floats: read-only / write-only / copy
        x = torch.randn(1 << 28, device=dev)
        y = torch.empty_like(x)
        for name, fn, nbytes in (("read(sum)", lambda: x.sum(), 4 << 28),
                                 ("write(fill)", lambda: y.fill_(1.0), 4 << 28),
                                 ("copy", lambda: y.copy_(x), 8 << 28)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.iters
            print(json.dumps({"case": name, "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9}), flush=True)
        return
    elif a.case == "mlp":
        # BASELINE config 2 gradients (784-1200-1200-10): exchange step latency
        import time

        sizes = [(784, 1200), (1200,), (1200, 1200), (1200,), (1200, 10), (10,)]
        gs = [torch.randn(s, device=dev) * 1e-3 for s in sizes]
        outs = [torch.empty_like(g) for g in gs]
        for graph in (False, True):
            kw = {"graph": True} if graph else {}
            try:
                ex = A.GradientExchange(spec, check="deferred", **kw)
            except TypeError:
                continue
            for _ in range(5):
                ex(gs, out=outs)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            for _ in range(a.iters):
                ex(gs, out=outs)
            e1.record()
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / a.iters * 1e6
            print(json.dumps({"case": "mlp_exchange", "graph": graph, "n": sum(g.numel() for g in gs),
                              "gpu_us_per_step": e0.elapsed_time(e1) / a.iters * 1e3,
                              "wall_us_per_step": wall}), flush=True)
        return
    elif a.case == "sweep":
        cases = [(f"2^{k}", [(1 << k,)]) for k in range(10, 31, 2)]
    else:
        raise SystemExit(f"unknown case {a.case}")
    for name, sizes in cases:
        n, res = run(sizes, spec, a.iters, dev)
        print(json.dumps({"case": name, "spec": a.spec, "n": n, **res}), flush=True)


if __name__ == "__main__":
    main()
