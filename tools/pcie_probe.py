"""PCIe reference numbers for the e2e line: pinned H2D alone, D2H alone, and
both directions concurrently (244 MB each, the C3 gradient size)."""
import json
import torch

n = 61_100_840
dev = torch.device("cuda", 0)
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, device=dev)
d_b = torch.empty(n, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
res = {}
for name in ("h2d", "d2h", "both"):
    for rep in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if name in ("h2d", "both"):
            s1.wait_event(e0)
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if name in ("d2h", "both"):
            s2.wait_event(e0)
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    res[name] = {"ms": ms, "GBps_per_direction": 4 * n / (ms * 1e-3) / 1e9}
print(json.dumps(res))
