import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, threading
from helpers import O, run_virtual_ranks
import paper_1511_04561_b200 as A
from paper_1511_04561_b200.exchange import CudaSegmentCodec
exec(open('tools/dbg_exchange2.py').read().split('res = run_virtual_ranks(nr, body)')[0])
res = run_virtual_ranks(nr, body)
enc2 = [s for s in log['r0'] if s[0]=='enc'][1]
_, ns, offs, idx, lay, xs, buf = enc2
np.savez('gpurun_out/round2_r0.npz', *xs)
L = 19168; B = L + 64
for trial in range(3):
    base = torch.zeros(L, device=dev)
    for o, x in zip(offs, xs): base[o:o+x.size] = torch.from_numpy(x)
    ts = [base[o:o+x.size] for o, x in zip(offs, xs)]
    out = torch.zeros(4*B, dtype=torch.uint8, device=dev)
    st_in = torch.zeros(1, dtype=torch.int32, device=dev)
    CudaSegmentCodec().encode(ts, offs, list(range(len(xs))), A.build_codebook(spec), out, 0, L, L, B, 0, 1, L+64, status_in=st_in)
    torch.cuda.synchronize(); mem = out.cpu().numpy()
    for t,(o,x) in enumerate(zip(offs, xs)):
        ref, s = O.encode(x, 'dynamic-tree', 'absmax')
        got = mem[o:o+x.size]; sc = np.frombuffer(mem[L+4*t:L+4*t+4].tobytes(), np.float32)[0]
        print('trial', trial, 'piece', t, 'n', x.size, 'ok', np.array_equal(got, ref), 'scale', sc, s)
