"""1-bit error-feedback quantizer timing (one GPU): onebit_quantize (stats +
apply launches) and onebit_decode on float32 gradients with a float64
residual, n = 2^20 .. 2^28.  CUDA events around the calls after warm-up
(the calls are asynchronous: sync=False); traffic per element: quantize
reads g (4 B) + residual (8 B) twice and writes residual (8 B) + 1/8 B of
bits = 28.1 B, decode writes 4 B (+1/8 B read)."""
import json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa

dev = torch.device("cuda", 0)
for k in (20, 24, 26, 28):
    n = 1 << k
    g = torch.randn(n, device=dev) * 1e-3
    st = A.OneBitState.zeros((n,), device=dev)
    for _ in range(3):
        q = A.onebit_quantize(g, st, sync=False)
        A.onebit_decode(q)
    torch.cuda.synchronize()
    tq, td = [], []
    for _ in range(5):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        q = A.onebit_quantize(g, st, sync=False)
        e1.record()
        A.onebit_decode(q)
        e2.record()
        torch.cuda.synchronize()
        tq.append(e0.elapsed_time(e1))
        td.append(e1.elapsed_time(e2))
    mq, md = float(np.median(tq)), float(np.median(td))
    print(json.dumps({"n": n, "quantize_us": mq * 1e3, "decode_us": md * 1e3,
                      "quantize_GBps": 28.125 * n / (mq * 1e-3) / 1e9, "decode_GBps": 4.125 * n / (md * 1e-3) / 1e9}),
          flush=True)
