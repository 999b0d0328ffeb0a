"""One per-block encode configuration for ncu: python tools/prof_blocked_one.py LOG2 BLOCK [REPS]."""
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa: E402

k, block = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda", 0)
x = torch.randn(1 << k, device=dev)
cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
for _ in range(reps):
    q = A.encode_buffer(x, cb, block_size=block, sync=False)
torch.cuda.synchronize()
q._finish()
print("ok")
