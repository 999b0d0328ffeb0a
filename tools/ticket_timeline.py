"""Per-CTA ticket timeline of one C3 encode launch (debug library only).

    python paper_1511_04561_b200/build.py --ticket-trace
    A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so [A8_PREMAX=1] python tools/ticket_timeline.py

Prints the launch span, the ramp (first ticket issued / first ticket done
per CTA), the tail (last ticket done per CTA), the service interval between
a CTA's consecutive tickets by kind, and the table switches' cost.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
assert os.environ.get("A8_LIB"), "set A8_LIB to the --ticket-trace build"

import paper_1511_04561_b200 as A  # noqa: E402
from paper_1511_04561_b200 import _native as N  # noqa: E402
from prof_codec import ALEXNET, run  # noqa: E402

KIND = {0: "A", 1: "E", 2: "B", 3: "F"}


def pct(a, q):
    return float(np.percentile(a, q)) if len(a) else float("nan")


def main():
    dev = torch.device("cuda", 0)
    lib = N.lib
    lib.a8_debug_switch_trace.restype = C.c_int
    lib.a8_debug_switch_trace.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    ntk = 1 << 17
    buf = (C.c_uint64 * (5 * ntk))()
    sw = (C.c_uint64 * (8 * (1 << 14)))()
    run(ALEXNET, A.parse_spec("dynamic-tree/absmax"), 4, dev)
    torch.cuda.synchronize()
    lib.a8_debug_switch_trace(sw, 1 << 14, 1)
    n, res = run(ALEXNET, A.parse_spec("dynamic-tree/absmax"), 1, dev)
    torch.cuda.synchronize()
    print("encode event time (median, trace build):", res["encode"])
    cnt = lib.a8_debug_switch_trace(sw, 1 << 14, 0)
    N.check(lib.a8_debug_ticket_trace(buf, C.c_int64(ntk)))
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(ntk, 5).astype(np.int64)
    used = tr[:, 0] > 0
    last = tr[used, 0].max()
    sel = np.where(used & (tr[:, 0] > last - 1_000_000))[0]
    t0 = tr[sel, 0].min()
    iss, done = (tr[sel, 0] - t0) / 1e3, (tr[sel, 1] - t0) / 1e3
    cta = tr[sel, 2] & 0xFFFFF
    kind = (tr[sel, 2] >> 40) & 0xFF
    print(f"tickets {len(sel)}, span {done.max():.1f} us")
    first_done = np.array([done[cta == c].min() for c in np.unique(cta)])
    last_done = np.array([done[cta == c].max() for c in np.unique(cta)])
    print(f"ramp: first ticket done per CTA p10/p50/p90 {pct(first_done,10):.1f}/{pct(first_done,50):.1f}/"
          f"{pct(first_done,90):.1f} us; tail: last done p10/p50/p90 {pct(last_done,10):.1f}/"
          f"{pct(last_done,50):.1f}/{pct(last_done,90):.1f} us")
    # service interval: time between a CTA's consecutive completions, by the later ticket's kind
    gaps = {k: [] for k in KIND}
    for c in np.unique(cta):
        m = np.where(cta == c)[0]
        o = m[np.argsort(done[m])]
        d = np.diff(done[o])
        for k, g in zip(kind[o][1:], d):
            gaps[int(k)].append(g)
    for k, g in gaps.items():
        if g:
            g = np.array(g)
            print(f"  {KIND[k]}: {len(g)} intervals, mean {g.mean():.2f} us, p50 {pct(g,50):.2f}, p90 {pct(g,90):.2f},"
                  f" p99 {pct(g,99):.2f}, sum {g.sum():.0f} us")
    s = np.frombuffer(sw, dtype=np.uint64).reshape(-1, 8).astype(np.int64)[:min(cnt, 1 << 14)]
    s = s[(s[:, 3] >= t0) & (s[:, 3] < t0 + 2_000_000)]
    modes = (s[:, 1] >> 24) & 0xFF
    for md, name in ((4, "prefetch"), (2, "copy"), (3, "build+pub"), (1, "local"), (0, "B-none")):
        r = s[modes == md]
        if len(r):
            print(f"  switch {name}: {len(r)} x mean {np.mean(r[:, 7] - r[:, 3]) / 1e3:.2f} us "
                  f"(sum {np.sum(r[:, 7] - r[:, 3]) / 1e3:.0f} us)")
            if md in (1, 3) and (r[:, 5] > 0).all() and (r[:, 6] > 0).all():
                print(f"    phases: thresholds {np.mean(r[:, 5] - r[:, 3]) / 1e3:.2f} fill "
                      f"{np.mean(r[:, 6] - r[:, 5]) / 1e3:.2f} end {np.mean(r[:, 7] - r[:, 6]) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
