timeout 900 python - <<'PY' 2>&1 | tail -30
import json, sys, torch
sys.path.insert(0, ".")
import bench, paper_1511_04561_b200 as A
class Nop:
    def __init__(self, i): pass
    def __enter__(self): return self
    def __exit__(self, *a): pass
    def summary(self): return {}
dev = torch.device("cuda", 0)
r = bench.codec_sweep(A, torch, dev, Nop)
for x in r["blocked"]: print(x["n"], x["block"], round(x["encode_ms"]*1e3,1), round(x["decode_ms"]*1e3,1), round(x["roundtrip_frac"],3))
PY
