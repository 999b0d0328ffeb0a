"""Phase stamps of one grid-barrier encode launch at config 3 (debug library only):
    A8_LIB=paper_1511_04561_b200/_lib_var/<trace build>/libapprox8_b200.so python tools/gb_trace.py
Per CTA: A pass end, barrier exit, first table ready, end (us from the first CTA's start)."""
import ctypes as C, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200 import _native as N  # noqa
dev = torch.device("cuda", 0)
grads = [torch.from_numpy(g).to(dev) for g in bench.alexnet_grads(0)]
outs = [torch.empty_like(g) for g in grads]
ex = A.GradientExchange(A.parse_spec("dynamic-tree/absmax"), check="sync")
for _ in range(4):
    ex(grads, out=outs)
torch.cuda.synchronize()
buf = (C.c_uint64 * (160 * 6))()
N.lib.a8_debug_gb_trace.argtypes = [C.c_void_p]
N.lib.a8_debug_gb_trace(buf)
t = np.array(buf, dtype=np.float64).reshape(160, 6)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t[:, :5] - t0) / 1e3
names = ["start", "A done", "barrier left", "kept done", "end"]
for i, n in enumerate(names):
    c = rel[:, i]
    print(f"{n:13s} min {c.min():7.2f} p50 {np.median(c):7.2f} p90 {np.percentile(c, 90):7.2f} max {c.max():7.2f}")
print("chunks per CTA", int(t[:, 5].min()), int(t[:, 5].max()), "ctas", len(t))
slow = np.argsort(rel[:, 1])[-5:]
print("slowest A passes (cta, chunks, A done):", [(int(i), int(t[i, 5]), round(rel[i, 1], 2)) for i in slow])
# structure of the end times: by CTA index (groups of 16) and by SM pair (b, b + G/2)
end = rel[:, 4]
print("end by CTA block of 16:", [round(float(end[i:i + 16].mean()), 1) for i in range(0, len(end), 16)])
ed = rel[:, 4] - rel[:, 2]
print("E duration by CTA block of 16:", [round(float(ed[i:i + 16].mean()), 1) for i in range(0, len(ed), 16)])
ad = rel[:, 1] - rel[:, 0]
print("A duration by CTA block of 16:", [round(float(ad[i:i + 16].mean()), 1) for i in range(0, len(ad), 16)])
