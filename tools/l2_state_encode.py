"""C3 encode time as a function of the L2 state it starts from (one B200):
after a 256 MB read (clean L2), after a 256 MB write (dirty L2), after the
step's decode (its 244 MB output partly dirty in L2), back to back."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_1511_04561_b200 as A  # noqa: E402
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan  # noqa: E402
from prof_codec import ALEXNET  # noqa: E402

dev = torch.device("cuda", 0)
xs = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in ALEXNET]
outs = [torch.empty_like(x) for x in xs]
plan = make_plan([x.numel() for x in xs], 1)
cb = A.build_codebook(A.parse_spec("dynamic-tree/absmax"))
codec = CudaSegmentCodec()
B = plan.allgather_block()
buf = torch.zeros(B, dtype=torch.uint8, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
idx = list(range(len(xs)))
big = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB


def enc():
    codec.encode(xs, plan.offs, idx, cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, 1, plan.flat + 4 * plan.status_slot)


def dec():
    codec.decode(outs, plan.offs, idx, cb, buf, 0, plan.flat, plan.flat, plan.flat, 0, B, 1, 1, plan.status_slot, 1, st)


pre = {"after 256 MB read": lambda: big.sum(), "after 256 MB write": lambda: big.fill_(1.0),
       "after decode": dec, "after encode": enc}
for _ in range(3):
    enc(); dec()
torch.cuda.synchronize()
for name, fn in pre.items():
    ts = []
    for _ in range(15):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); enc(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"encode {name}: {np.median(ts):.1f} us")
ts = []
for _ in range(15):
    enc()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dec(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"decode after encode: {np.median(ts):.1f} us")
