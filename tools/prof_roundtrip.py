"""Fused round trip (a8_roundtrip, one kernel) vs encode + decode (two
kernels), graph-captured events, L2 flushed per rep; the MLP seam sizes."""
import ctypes as C, json, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200 import _native as N  # noqa
from paper_1511_04561_b200.codecs import workspace, round16  # noqa

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for label in ("dynamic-tree/absmax", "mantissa/decade+2"):
    spec = A.parse_spec(label)
    cb = A.build_codebook(spec)
    book, lut = cb.device_tables(dev)
    for n in (128 * 1200, 784 * 1200, 1 << 20, 1200 * 1200, 1 << 22):
        x = torch.randn(n, device=dev)
        out = torch.empty_like(x)
        codes = torch.empty(n, dtype=torch.uint8, device=dev)
        meta = torch.zeros(2, dtype=torch.int32, device=dev)
        s = torch.cuda.Stream(dev)
        ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]

        def step():
            st = torch.cuda.current_stream(dev).cuda_stream
            ws = workspace(dev, st, 1)
            seg = N.EncSeg(x.data_ptr(), n, 0, 0, 0)
            ev[0].record()
            outs = (C.c_void_p * 1)(out.data_ptr())
            N.check(N.lib.a8_roundtrip(C.byref(seg), outs, 1, book.data_ptr(), spec.norm_code,
                                       None if lut is None else lut.data_ptr(), meta.data_ptr() + 4, meta.data_ptr(),
                                       ws.data_ptr(), ws.numel(), st))
            ev[1].record()
            lay = N.Layout(codes.data_ptr(), meta.data_ptr() + 4, round16(n), round16(n), 0, 0, 1, 0)
            N.check(N.lib.a8_encode(C.byref(seg), 1, book.data_ptr(), spec.norm_code,
                                    None if lut is None else lut.data_ptr(), lay, ws.data_ptr(), ws.numel(), None,
                                    meta.data_ptr(), st))
            dseg = N.DecSeg(out.data_ptr(), n, 0, 0, 0)
            N.check(N.lib.a8_decode(C.byref(dseg), 1, book.data_ptr(), lay, 1, 0, -1, 0, None, ws.data_ptr(),
                                    ws.numel(), st))
            ev[2].record()

        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        a, b = [], []
        for _ in range(7):
            flush.fill_(1)
            g.replay()
            torch.cuda.synchronize()
            a.append(ev[0].elapsed_time(ev[1]))
            b.append(ev[1].elapsed_time(ev[2]))
        print(json.dumps({"spec": label, "n": n, "fused_us": float(np.median(a)) * 1e3,
                          "encode_plus_decode_us": float(np.median(b)) * 1e3}), flush=True)
