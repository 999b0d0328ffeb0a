# per-block codec at 2^30 (B = 4096 / 1024), current build vs git stash of the previous
timeout 900 python - <<'PY'
import json, sys, torch
sys.path.insert(0, ".")
import bench, paper_1511_04561_b200 as A
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def tg(fn, reps=7):
    s = torch.cuda.Stream(dev); s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream(dev).wait_stream(s); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s): fn()
    ts = []
    for _ in range(reps):
        flush.zero_(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    import numpy as np; return float(np.median(ts))
cb = A.build_codebook(A.parse_spec("dynamic-tree/absmax"))
x = torch.randn(1 << 30, device=dev)
for b in (4096, 2048, 1024):
    box = {}
    t = tg(lambda: box.__setitem__("q", A.encode_buffer(x, cb, sync=False, block_size=b)))
    print(b, "encode us", round(t * 1e3, 1), "frac", round(5 * 2**30 / (t * 1e-3) / 1e9 / 6543.1, 3))
PY
