# Producer-fused max + one-pass encode: GPU tests and the premax sweep numbers.
mkdir -p gpurun_out
python -c "import paper_1511_04561_b200._native as N, ctypes as C; a=C.c_int(); b=C.c_int(); c=C.c_int(); N.lib.a8_device_info(0, C.byref(a), C.byref(b), C.byref(c)); print('sms', a.value, 'enc_occ', b.value, 'dec_occ', c.value)"
timeout 900 python -m pytest tests/test_gpu_premax.py -x -q 2>&1 | tail -15; echo premax_tests=$?
timeout 900 python - <<'PY' 2>&1 | tail -30
import json, sys, torch
sys.path.insert(0, ".")
import bench, paper_1511_04561_b200 as A
dev = torch.device("cuda", 0)
import numpy as np
# only the premax part of the sweep
src = open("bench.py").read()
out = {}
class Nop:
    def __init__(self, i): pass
    def __enter__(self): return self
    def __exit__(self, *a): pass
    def summary(self): return {}
# run the full sweep function body but only print the premax part
r = bench.codec_sweep(A, torch, dev, Nop)
print(json.dumps(r["premax"], indent=1))
print(json.dumps({k: [(x["n"], x["spec"], round(x["encode_ms"]*1e3,1), round(x["decode_ms"]*1e3,1)) for x in v] for k, v in r.items() if isinstance(v, list)}))
PY
