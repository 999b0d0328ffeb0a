"""Table-switch timeline of one C3 encode launch (debug library only).

    python paper_1511_04561_b200/build.py --ticket-trace
    A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so python tools/switch_trace.py

Per segment: when its A pass ended, when its table was published (the B
build), when its E tickets were issued, and how the CTAs got the table
(4 = producer prefetch, 2 = copy, 3 = build + publish, 1 = local build,
0 = B without work) with the time each cost.
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

MODES = {0: "B-none", 1: "local", 2: "copy", 3: "build+pub", 4: "prefetch"}


def main():
    dev = torch.device("cuda", 0)
    lib = N.lib
    lib.a8_debug_switch_trace.restype = C.c_int
    lib.a8_debug_switch_trace.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    ntk = 1 << 17
    buf = (C.c_uint64 * (5 * ntk))()
    sw = (C.c_uint64 * (8 * (1 << 14)))()
    n, res = run(ALEXNET, A.parse_spec("dynamic-tree/absmax"), 4, dev)
    torch.cuda.synchronize()
    lib.a8_debug_switch_trace(sw, 1 << 14, 1)  # reset the counter
    n, res = run(ALEXNET, A.parse_spec("dynamic-tree/absmax"), 1, dev)  # 3 warm-up + 2 timed launches
    torch.cuda.synchronize()
    cnt = lib.a8_debug_switch_trace(sw, 1 << 14, 0)
    N.check(lib.a8_debug_ticket_trace(buf, C.c_int64(ntk)))
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(ntk, 5).astype(np.int64)
    used = tr[:, 0] > 0
    last = tr[used, 0].max()
    sel = used & (tr[:, 0] > last - 1_000_000)
    t0 = tr[sel, 0].min()
    kinds = (tr[:, 2] >> 40) & 0xFF
    segs_of = (tr[:, 2] >> 20) & 0xFFFFF
    s = np.frombuffer(sw, dtype=np.uint64).reshape(-1, 8).astype(np.int64)[:min(cnt, 1 << 14)]
    s = s[(s[:, 3] >= t0) & (s[:, 3] < t0 + 2_000_000)]
    print(f"kernel span {(tr[sel, 1].max() - t0) / 1e3:.1f} us, switches logged {len(s)}")
    for sg in sorted(set(segs_of[sel].tolist())):
        m = sel & (segs_of == sg)
        a = m & (kinds == 0)
        e = m & (kinds == 1)
        if not e.any():
            continue
        rows = s[s[:, 2] == sg]
        pub = rows[((rows[:, 1] >> 24) & 0xFF) == 3]
        pub_t = (pub[:, 7].min() - t0) / 1e3 if len(pub) else float("nan")
        line = (f"seg {sg:2d}: A issue {(tr[a, 0].min() - t0) / 1e3:6.1f}..{(tr[a, 0].max() - t0) / 1e3:6.1f} "
                f"done {(tr[a, 1].max() - t0) / 1e3:6.1f} | published {pub_t:6.1f} | E issue "
                f"{(tr[e, 0].min() - t0) / 1e3:6.1f}..{(tr[e, 0].max() - t0) / 1e3:6.1f} |")
        for md in (4, 2, 3, 1, 0):
            r = rows[((rows[:, 1] >> 24) & 0xFF) == md]
            if len(r):
                line += f" {MODES[md]} {len(r)}x{np.mean(r[:, 7] - r[:, 3]) / 1e3:.2f}us"
        print(line)
    # where builds spend their time
    b = s[((s[:, 1] >> 24) & 0xFF) == 3]
    if len(b):
        d = np.diff(b[:, 3:8], axis=1) / 1e3
        print("build+pub phases (us): wait-max %.2f thresholds %.2f fill %.2f publish %.2f" % tuple(d.mean(axis=0)))
    loc = s[((s[:, 1] >> 24) & 0xFF) == 1]
    if len(loc):
        d = np.diff(loc[:, 3:8], axis=1) / 1e3
        print("local build phases (us): wait-max %.2f thresholds %.2f fill %.2f end %.2f" % tuple(d.mean(axis=0)))


if __name__ == "__main__":
    main()
