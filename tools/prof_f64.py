"""float64-input encode (a8_encode_f64) timing on one GPU: the reference's
DP/MP seams feed float64 (mlp.py:330).  CUDA events around the call after
warm-up; algorithmic bytes 8 B read + 1 B written per element."""
import json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa

dev = torch.device("cuda", 0)
for label in ("dynamic-tree/absmax", "mantissa/decade+2"):
    cb = A.build_codebook(A.parse_spec(label))
    for k in (20, 24, 26):
        n = 1 << k
        x = torch.randn(n, device=dev, dtype=torch.float64) * 0.01
        for _ in range(3):
            A.encode_buffer(x, cb, sync=False)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            A.encode_buffer(x, cb, sync=False)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(json.dumps({"spec": label, "n": n, "encode_us": ms * 1e3, "GBps": 9.0 * n / (ms * 1e-3) / 1e9}), flush=True)
