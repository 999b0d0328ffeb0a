"""Per-ticket timeline of one encode launch (debug library only).

    python paper_1511_04561_b200/build.py --ticket-trace
    A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so python tools/ticket_trace.py [--case alexnet|single]

Prints, per 2 us window, the tickets completed by kind and the DRAM-side bytes
they stand for, plus per-segment phase times (first issue .. last done of its
A and E tickets).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
assert os.environ.get("A8_LIB"), "set A8_LIB to the --ticket-trace build"

import paper_1511_04561_b200 as A  # noqa: E402
from paper_1511_04561_b200 import _native as N  # noqa: E402
import prof_codec  # noqa: E402
from prof_codec import ALEXNET, run  # noqa: E402

KIND = {0: "A", 1: "E", 2: "B", 3: "F"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="alexnet")
    ap.add_argument("--out", default="gpurun_out/ticket_trace.json")
    ap.add_argument("--spec", default="dynamic-tree/absmax")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sizes = ALEXNET if a.case == "alexnet" else [(1 << 26,)]
    prof_codec.TRACE = True  # also read the per-segment build stamps
    n, res = run(sizes, A.parse_spec(a.spec), 5, dev)  # last call = the traced one
    torch.cuda.synchronize()
    ntk = 1 << 17
    buf = (C.c_uint64 * (5 * ntk))()
    N.check(N.lib.a8_debug_ticket_trace(buf, C.c_int64(ntk)))
    tr = np.frombuffer(buf, dtype=np.uint64).reshape(ntk, 5).astype(np.int64)
    used = tr[:, 0] > 0
    t0 = tr[used, 0].min()
    # only tickets of the last launch: issue times within 1 ms of the latest
    last = tr[used, 0].max()
    sel = used & (tr[:, 0] > last - 1_000_000)
    idx = np.nonzero(sel)[0]
    t0 = tr[idx, 0].min()
    rows = []
    for t in idx:
        iss, done, meta, known, free = tr[t]
        rows.append({"t": int(t), "kind": KIND.get(int(meta >> 40), "?"), "seg": int((meta >> 20) & 0xFFFFF),
                     "cta": int(meta & 0xFFFFF), "issue_us": (iss - t0) / 1e3, "done_us": (done - t0) / 1e3,
                     "known_us": (known - t0) / 1e3, "free_us": (free - t0) / 1e3})
    segs = {}
    for r in rows:
        d = segs.setdefault((r["seg"], r["kind"]), [1e9, 0, 0])
        d[0] = min(d[0], r["issue_us"])
        d[1] = max(d[1], r["done_us"])
        d[2] += 1
    print(json.dumps({"case": a.case, "n": n, "encode_ms": res["encode"]["ms"], "tickets": len(rows)}))
    print(json.dumps(res.get("trace")))
    for (sg, k), (b, e, c) in sorted(segs.items(), key=lambda kv: kv[1][0]):
        print(f"seg {sg:3d} {k}: {c:6d} tickets  issue {b:8.2f} .. done {e:8.2f} us")
    end = max(r["done_us"] for r in rows)
    W = 2.0
    nb = int(end / W) + 1
    hist = {k: np.zeros(nb) for k in "AEF"}
    lat = np.zeros(nb)
    cnt = np.zeros(nb)
    for r in rows:
        if r["kind"] in hist:
            b = int(r["done_us"] / W)
            hist[r["kind"]][b] += 1
            lat[b] += r["done_us"] - r["issue_us"]
            cnt[b] += 1
    print(" window_us   A_done  E_done  F_done  GB/s(A:4B,E:5B/elem)  mean issue->done us")
    for b in range(nb):
        gbs = (hist["A"][b] * 4096 * 4 + hist["E"][b] * 4096 * 5) / (W * 1e-6) / 1e9
        print(f"{b * W:7.1f}  {int(hist['A'][b]):7d} {int(hist['E'][b]):7d} {int(hist['F'][b]):7d}  {gbs:9.0f}  "
              f"{lat[b] / max(cnt[b], 1):8.2f}")
    fl = (C.c_uint64 * (32 * 512 * 4))()
    N.check(N.lib.a8_debug_flush_trace(fl))
    fl = np.frombuffer(fl, dtype=np.uint64).reshape(32, 512, 4).astype(np.int64)
    for sg in range(32):
        v = fl[sg][fl[sg, :, 0] > last - 1_000_000]
        if len(v) == 0:
            continue
        f0, f1 = (v[:, 0] - t0) / 1e3, (v[:, 1] - t0) / 1e3
        lastc = v[v[:, 2] > 0]
        print(f"flush seg {sg:3d}: {len(v)} CTAs, start {f0.min():7.2f}..{f0.max():7.2f}  atom rtt mean "
              f"{(f1 - f0).mean():5.2f} max {(f1 - f0).max():5.2f}  last contributor amax back "
              f"{((lastc[:, 2] - t0) / 1e3).tolist()}")
    Path(a.out).parent.mkdir(exist_ok=True)
    Path(a.out).write_text(json.dumps(rows))


if __name__ == "__main__":
    main()
