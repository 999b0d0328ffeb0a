import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, torch
from helpers import O, run_virtual_ranks
import paper_1511_04561_b200 as A
SMALL = [(40, 30), (1,), (17,), (0,), (300,), (4, 4, 4), (5000,), (70000,)]
def grads(rank, sizes, seed=0, sigma=1e-2):
    rng = np.random.default_rng(seed * 1000 + rank)
    return [rng.normal(0.0, sigma, size=s).astype(np.float32) for s in sizes]
dev=torch.device('cuda',0)
for nr, mode, spec in [(4,'two_round',A.DataTypeSpec('dynamic-tree','absmax')),(3,'allgather',A.DataTypeSpec('linear','absmax')),(3,'two_round',A.DataTypeSpec('linear','absmax'))]:
    def body(rank, comm):
        ex = A.GradientExchange(spec, mode=mode, op='avg', check='sync', comm=comm)
        ts = [torch.from_numpy(g).to(dev) for g in grads(rank, SMALL, 4 if nr==3 else 0)]
        ex(ts); torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]
    res = run_virtual_ranks(nr, body)
    g = [grads(r, SMALL, 4 if nr==3 else 0) for r in range(nr)]
    fn = O.exchange_allgather if mode == 'allgather' else O.exchange_two_round
    want = fn(g, spec.kind.value, spec.normalization.value, spec.decades, 'avg')
    for r in range(nr):
        for t,(a,b) in enumerate(zip(res[r], want)):
            a=a.ravel(); b=b.ravel()
            if a.tobytes()!=b.tobytes():
                bad=np.nonzero(a!=b)[0]
                print(nr,mode,spec.label(),'rank',r,'tensor',t,'n',a.size,'nbad',bad.size,'first',bad[:5], a[bad[:3]], b[bad[:3]])
