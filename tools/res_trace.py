"""Phase stamps of one resident encode launch (debug library only):
    A8_LIB=paper_1511_04561_b200/_lib_trace/libapprox8_b200.so python tools/res_trace.py"""
import ctypes as C, json, sys
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1511_04561_b200 as A  # noqa
from paper_1511_04561_b200 import _native as N  # noqa
from prof_codec import run  # noqa
dev = torch.device("cuda", 0)
for name, sizes in (("mlp", [(784, 1200), (1200,), (1200, 1200), (1200,), (1200, 10), (10,)]), ("c5", [(128, 512)]), ("c1", [(1 << 20,)]), ("tiny", [(1024,)])):
    run(sizes, A.parse_spec("dynamic-tree/absmax"), 3, dev)
    torch.cuda.synchronize()
    lib = N.lib
    lib.a8_debug_res_trace.argtypes = [C.c_void_p]
    buf = (C.c_uint64 * 16)()
    lib.a8_debug_res_trace(buf)
    t0 = buf[0]
    print(name, "cta0:", [round((buf[i] - t0) / 1e3, 2) for i in range(6)],
          "last:", [round((buf[8 + i] - t0) / 1e3, 2) for i in range(6)])
