import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch, threading
from helpers import O, run_virtual_ranks
import paper_1511_04561_b200 as A
from paper_1511_04561_b200.exchange import CudaSegmentCodec
SMALL = [(40, 30), (1,), (17,), (0,), (300,), (4, 4, 4), (5000,), (70000,)]
def grads(rank, sizes, seed=0, sigma=1e-2):
    rng = np.random.default_rng(seed * 1000 + rank)
    return [rng.normal(0.0, sigma, size=s).astype(np.float32) for s in sizes]
dev=torch.device('cuda',0)
spec=A.DataTypeSpec('dynamic-tree','absmax'); nr=4
log={}
class Rec(CudaSegmentCodec):
    def encode(self, xs, flat_offs, scale_idx, cb, buf, *a, **k):
        super().encode(xs, flat_offs, scale_idx, cb, buf, *a, **k); torch.cuda.synchronize()
        r=threading.current_thread().name
        log.setdefault(r,[]).append(('enc',[x.numel() for x in xs], list(flat_offs), list(scale_idx), a[:6], [x.cpu().numpy().copy() for x in xs], buf.cpu().numpy().copy()))
    def decode(self, outs, flat_offs, scale_idx, cb, buf, *a, **k):
        super().decode(outs, flat_offs, scale_idx, cb, buf, *a, **k); torch.cuda.synchronize()
        r=threading.current_thread().name
        log.setdefault(r,[]).append(('dec',[x.numel() for x in outs], list(flat_offs), list(scale_idx), a[:8], [x.cpu().numpy().copy() for x in outs]))
def body(rank, comm):
    threading.current_thread().name=f"r{rank}"
    ex = A.GradientExchange(spec, mode='two_round', op='avg', check='sync', codec=Rec(), comm=comm)
    ts = [torch.from_numpy(g).to(dev) for g in grads(rank, SMALL)]
    ex(ts); torch.cuda.synchronize()
    return [t.cpu().numpy() for t in ts]
res = run_virtual_ranks(nr, body)
for step in log['r0']:
    if step[0]=='enc':
        _, ns, offs, idx, lay, xs, buf = step
        print('ENC ns',ns,'offs',offs,'idx',idx,'lay',lay)
        codes_off, scales_off, L, stride = lay[0], lay[1], lay[2], lay[3]
        for n,o,x in zip(ns,offs,xs):
            e=np.arange(n)+o; c=buf[codes_off + (e//L)*stride + e%L]
            ref,s=O.encode(x,'dynamic-tree','absmax')
            print('   seg n',n,'codes ok',np.array_equal(c,ref),'nz',int((c!=0).sum()),'refnz',int((ref!=0).sum()))
    else:
        _, ns, offs, idx, lay, outs = step
        print('DEC ns',ns,'offs',offs,'idx',idx,'lay',lay, 'out nonzero', [int((o!=0).sum()) for o in outs])
# dump the failing round-2 input of rank 0 and replay single-threaded
enc2 = [s for s in log['r0'] if s[0]=='enc'][1]
x6 = enc2[5][6]
np.save('gpurun_out/x6.npy', x6)
cb = A.build_codebook(spec)
q = A.encode_buffer(torch.from_numpy(x6).to(dev), cb)
ref, s = O.encode(x6, 'dynamic-tree', 'absmax')
print('replay single encode_buffer ok:', np.array_equal(q.codes.cpu().numpy(), ref), 'scale', q.scale, s)
for _ in range(3):
    res = run_virtual_ranks(nr, body)
