"""1-bit exchange over the config-3 gradients (N = 1), for ncu launch lists."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda", 0)
ts = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in bench.ALEXNET]
outs = [torch.empty_like(t) for t in ts]
ex = A.GradientExchange("onebit", check="none")
for _ in range(3):
    ex(ts, out=outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    ex(ts, out=outs)
e1.record()
torch.cuda.synchronize()
print("eager step us", e0.elapsed_time(e1) / 10 * 1e3)
