mkdir -p gpurun_out
timeout 900 python - <<'PY' 2>&1 | tail -40
import json, sys, torch
sys.path.insert(0, ".")
import bench, paper_1511_04561_b200 as A
class Nop:
    def __init__(self, i): pass
    def __enter__(self): return self
    def __exit__(self, *a): pass
    def summary(self): return {}
dev = torch.device("cuda", 0)
src = bench.codec_sweep.__code__
r = bench.codec_sweep(A, torch, dev, Nop)
print(json.dumps(r["premax"], indent=1))
PY
