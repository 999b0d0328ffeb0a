"""Per-block codec timing (graph-captured kernel events, L2 flushed per rep)."""
import json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200 import _native as N  # noqa

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
book, _ = cb.device_tables(dev)
for k in (20, 22, 24, 26, 28, 30):
    n = 1 << k
    x = torch.randn(n, device=dev)
    out = torch.empty_like(x)
    for block in (1024, 4096):
        nb = -(-n // block)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        sc = torch.empty(nb, device=dev)
        st = torch.empty(1, dtype=torch.int32, device=dev)
        s = torch.cuda.Stream(dev)
        ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]

        def step():
            stream = torch.cuda.current_stream(dev).cuda_stream
            ev[0].record()
            N.check(N.lib.a8_encode_blocked(x.data_ptr(), n, block, book.data_ptr(), codes.data_ptr(), sc.data_ptr(),
                                            st.data_ptr(), stream))
            ev[1].record()
            N.check(N.lib.a8_decode_blocked(codes.data_ptr(), n, block, sc.data_ptr(), book.data_ptr(), out.data_ptr(),
                                            stream))
            ev[2].record()

        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        e, d = [], []
        for _ in range(7):
            flush.fill_(1)
            g.replay()
            torch.cuda.synchronize()
            e.append(ev[0].elapsed_time(ev[1]))
            d.append(ev[1].elapsed_time(ev[2]))
        em, dm = float(np.median(e)), float(np.median(d))
        print(json.dumps({"n": n, "log2": k, "block": block, "encode_us": em * 1e3, "decode_us": dm * 1e3,
                          "encode_GBps": (5.0 * n + 4 * nb) / (em * 1e-3) / 1e9,
                          "decode_GBps": (5.0 * n + 4 * nb) / (dm * 1e-3) / 1e9}), flush=True)
