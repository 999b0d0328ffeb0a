"""The callers either side of the codec on the GPU.

* model-parallel FC (BASELINE config 5): 8-bit activation all-gather forward,
  8-bit partial error-signal sum backward, N virtual ranks on one GPU, exact
  against the composed oracle;
* LocalExchange (N replicas in one process) exact against the oracle;
* data-parallel MLP training (BASELINE config 2 shape) with the 8-bit
  exchange: final test error within 1 pp of 32-bit training over 3 seeds
  (the reference's parity criterion, test_acceptance.py:152-156).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O, run_virtual_ranks

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_model_parallel_fc_config5(nranks, cuda):
    rng = np.random.default_rng(nranks)
    x = torch.from_numpy(rng.normal(0, 0.02, size=(128, 4096)).astype(np.float32)).to(cuda)
    w = torch.from_numpy(rng.normal(0, 0.02, size=(4096, 4096)).astype(np.float32)).to(cuda)
    dy = torch.from_numpy(rng.normal(0, 1e-3, size=(128, 4096)).astype(np.float32)).to(cuda)
    k = 4096 // nranks
    spec = A.DataTypeSpec("dynamic-tree", "absmax")

    def body(rank, comm):
        fc = A.ModelParallelFC(w[:, rank * k:(rank + 1) * k].contiguous(), spec, comm=comm)
        y = fc.forward(x)
        y_r = (x @ fc.w).cpu().numpy()
        dx_r = (dy[:, rank * k:(rank + 1) * k] @ fc.w.t()).cpu().numpy()
        dx, dw = fc.backward(dy)
        torch.cuda.synchronize()
        return y.cpu().numpy(), dx.cpu().numpy(), y_r, dx_r

    res = run_virtual_ranks(nranks, body)
    y_want = np.concatenate([O.roundtrip(res[r][2], "dynamic-tree", "absmax") for r in range(nranks)], axis=1)
    dx_want = O.exchange_allgather([[res[r][3]] for r in range(nranks)], "dynamic-tree", "absmax", op="sum")[0]
    for r in range(nranks):
        assert res[r][0].tobytes() == y_want.tobytes(), r
        assert res[r][1].tobytes() == dx_want.tobytes(), r


def test_local_exchange_matches_oracle(cuda):
    rng = np.random.default_rng(3)
    shapes = [(784, 1200), (1200,), (1200, 1200), (1200,), (1200, 10), (10,)]
    for nrep in (1, 2, 3, 8):
        g = [[rng.normal(0, 1e-3, size=s).astype(np.float32) for s in shapes] for _ in range(nrep)]
        for op in ("avg", "sum"):
            out = A.LocalExchange(A.DataTypeSpec("dynamic-tree", "absmax"), op=op)(
                [[torch.from_numpy(t).to(cuda) for t in rep] for rep in g])
            want = O.exchange_allgather(g, "dynamic-tree", "absmax", op=op)
            for a, b in zip(out, want):
                assert a.cpu().numpy().tobytes() == b.tobytes(), (nrep, op)


def _dataset(seed, n_train=8000, n_test=4000):
    """Synthetic 10-class, 784-feature task (digit-like prototypes + noise)."""
    rng = np.random.default_rng(seed)
    protos = rng.uniform(0, 1, size=(10, 784)) * (rng.uniform(size=(10, 784)) < 0.3)
    def draw(n):
        y = rng.integers(0, 10, size=n)
        x = protos[y] + rng.normal(0, 0.35, size=(n, 784))
        return np.clip(x, 0, 1).astype(np.float32), y
    return draw(n_train), draw(n_test)


def _train(seed, spec, replicas=2, epochs=3, batch=128, dev="cuda"):
    """DP training of 784-1200-1200-10 (ReLU, softmax, RMSProp as mlp.py:371-375):
    each replica takes a batch of 128, gradients are exchanged (8-bit when
    `spec` is set, exact fp32 average otherwise), all replicas stay identical."""
    (xtr, ytr), (xte, yte) = _dataset(seed)
    torch.manual_seed(seed)
    sizes = (784, 1200, 1200, 10)
    params = []
    for a, b in zip(sizes, sizes[1:]):
        lim = (6.0 / (a + b)) ** 0.5
        params += [torch.empty(a, b, device=dev).uniform_(-lim, lim), torch.zeros(b, device=dev)]
    acc = [torch.zeros_like(p) for p in params]
    lr, decay, eps = 1e-3, 0.9, 1e-8
    ex = A.LocalExchange(spec) if spec is not None else None
    xtr_t, ytr_t = torch.from_numpy(xtr).to(dev), torch.from_numpy(ytr).to(dev)
    gen = np.random.default_rng(seed + 1)
    for _ in range(epochs):
        order = gen.permutation(len(xtr))
        for s in range(0, len(order) - replicas * batch + 1, replicas * batch):
            grads = []
            for r in range(replicas):
                idx = torch.from_numpy(order[s + r * batch:s + (r + 1) * batch]).to(dev)
                ps = [p.detach().requires_grad_(True) for p in params]
                h = xtr_t[idx]
                for l in range(3):
                    h = h @ ps[2 * l] + ps[2 * l + 1]
                    if l < 2:
                        h = torch.relu(h)
                loss = torch.nn.functional.cross_entropy(h, ytr_t[idx])
                grads.append([g.contiguous() for g in torch.autograd.grad(loss, ps)])
            if ex is not None:
                g = ex(grads)
            else:
                g = [sum(gr[i] for gr in grads) / replicas for i in range(len(params))]
            with torch.no_grad():
                for p, a, gi in zip(params, acc, g):
                    a.mul_(decay).add_((1 - decay) * gi * gi)
                    p.sub_(lr * gi / torch.sqrt(a + eps))
    with torch.no_grad():
        h = torch.from_numpy(xte).to(dev)
        for l in range(3):
            h = h @ params[2 * l] + params[2 * l + 1]
            if l < 2:
                h = torch.relu(h)
        return float((h.argmax(1).cpu().numpy() != yte).mean())


def test_dp_training_parity_config2(cuda):
    diffs = []
    for seed in (0, 1, 2):
        e32 = _train(seed, None)
        e8 = _train(seed, A.DataTypeSpec("dynamic-tree", "absmax"))
        diffs.append(100.0 * (e8 - e32))
        assert e32 < 0.2, e32  # the task is learnable in 3 epochs
    assert all(abs(d) < 1.0 for d in diffs), diffs


def _ddp_nccl_worker(port, q):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        spec = A.DataTypeSpec("dynamic-tree", "absmax")
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(), torch.nn.Linear(128, 10)).to(dev)
        ref = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(), torch.nn.Linear(128, 10)).to(dev)
        ref.load_state_dict(model.state_dict())
        ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[0])
        ddp.register_comm_hook(A.DDPHookState(spec, check="sync"), A.a8_comm_hook)
        x = torch.randn(32, 64, device=dev)
        y = torch.randn(32, 10, device=dev)
        torch.nn.functional.mse_loss(ddp(x), y).backward()
        torch.nn.functional.mse_loss(ref(x), y).backward()
        ok = True
        for p, r in zip(model.parameters(), ref.parameters()):
            want = O.roundtrip(r.grad.cpu().numpy(), "dynamic-tree", "absmax")  # N = 1: exchange == round trip
            ok &= p.grad.cpu().numpy().tobytes() == want.tobytes()
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_nccl_single_rank(cuda):
    """The DDP hook on the GPU with NCCL: a real DistributedDataParallel
    bucket goes through the sm_100a codec; at one rank every parameter's
    gradient equals the reference round trip of its local gradient."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_ddp_nccl_worker, args=(port, q))
    p.start()
    p.join(timeout=300)
    assert q.get(timeout=5) is True
