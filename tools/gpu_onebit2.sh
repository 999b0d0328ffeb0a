timeout 900 python -m pytest tests/test_gpu_onebit.py tests/test_gpu_exchange.py -q -k "onebit" 2>&1 | tail -3
python tools/prof_onebit_c3.py
timeout 900 python - <<'PY' 2>&1 | tail -3
import json, sys, torch
sys.path.insert(0, ".")
import bench, paper_1511_04561_b200 as A
class Nop:
    def __init__(self, i): pass
    def __enter__(self): return self
    def __exit__(self, *a): pass
    def summary(self): return {}
import types
dev = torch.device("cuda", 0)
r = bench.codec_sweep(A, torch, dev, Nop)
print(json.dumps(r["onebit_c3"]))
PY
