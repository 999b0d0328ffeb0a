"""Exchange orchestration on CPU: layouts, collectives, status propagation.

The codec work is done by the test-only ``NumpyCodec`` (the oracle behind the
C ABI's byte layout), so these tests check the product's slab layouts and
collective sequence -- allgather and two_round, avg and sum -- against the
composed exchange oracles, with real ``torch.distributed`` gloo ranks
(world_size 2) and with thread-based virtual ranks (world_size 2..5).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import NumpyCodec, NumpyOneBitCodec, O, run_virtual_ranks

import paper_1511_04561_b200 as A

SIZES = [(40, 30), (1,), (17,), (0,), (300,), (4, 4, 4), (1000,)]


def grads_for(rank, sizes=SIZES, seed=0, scale=1.0):
    rng = np.random.default_rng(seed * 1000 + rank)
    return [(rng.normal(size=s) * scale * (1 + i)).astype(np.float32) for i, s in enumerate(sizes)]


def expected(nranks, spec, mode, op, sizes=SIZES, seed=0):
    g = [grads_for(r, sizes, seed) for r in range(nranks)]
    fn = O.exchange_allgather if mode == "allgather" else O.exchange_two_round
    return fn(g, spec.kind.value, spec.normalization.value, spec.decades, op)


SPECS = [A.DataTypeSpec("dynamic-tree", "absmax"), A.DataTypeSpec("mantissa", "decade", 1),
         A.DataTypeSpec("linear", "absmax")]


@pytest.mark.parametrize("nranks", [2, 3, 5])
@pytest.mark.parametrize("mode", ["allgather", "two_round"])
@pytest.mark.parametrize("op", ["avg", "sum"])
def test_virtual_ranks_match_oracle(nranks, mode, op):
    spec = SPECS[nranks % len(SPECS)]

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode=mode, op=op, check="sync", codec=NumpyCodec(spec), comm=comm)
        ts = [torch.from_numpy(g) for g in grads_for(rank)]
        ex(ts)
        return [t.numpy().copy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    want = expected(nranks, spec, mode, op)
    for r in range(nranks):
        for a, b in zip(res[r], want):
            assert a.shape == b.shape
            assert np.array_equal(a, b), (r, mode, op)


@pytest.mark.parametrize("mode", ["allgather", "two_round"])
def test_nonfinite_on_one_rank_raises_on_all(mode):
    spec = SPECS[0]

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode=mode, check="sync", codec=NumpyCodec(spec), comm=comm)
        ts = [torch.from_numpy(g) for g in grads_for(rank)]
        if rank == 1:
            ts[4][7] = float("nan")
        try:
            ex(ts)
        except A.InputError:
            return "raised"
        return "ok"

    assert run_virtual_ranks(3, body) == ["raised"] * 3


def test_deferred_check_raises_on_next_call():
    spec = SPECS[0]

    def body(rank, comm):
        ex = A.GradientExchange(spec, check="deferred", codec=NumpyCodec(spec), comm=comm)
        ts = [torch.from_numpy(g) for g in grads_for(rank)]
        ts[0][0, 0] = float("inf")
        ex(ts)  # returns; status pending
        try:
            ex([torch.from_numpy(g) for g in grads_for(rank)])
        except A.InputError:
            return "raised"
        return "ok"

    assert run_virtual_ranks(2, body) == ["raised"] * 2


# ---------------------------------------------------------------------------
# real torch.distributed ranks (gloo, world_size 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, mode, op, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = SPECS[0]
        ex = A.GradientExchange(spec, mode=mode, op=op, check="sync", codec=NumpyCodec(spec))
        ts = [torch.from_numpy(g) for g in grads_for(rank)]
        ex(ts)
        ok = all(np.array_equal(t.numpy(), w) for t, w in zip(ts, expected(world, spec, mode, op)))
        # DDP-style hook path: bucket of views into one flat buffer
        flat = torch.cat([torch.from_numpy(g).reshape(-1) for g in grads_for(rank, seed=3)])
        views, pos = [], 0
        for s in SIZES:
            n = int(np.prod(s))
            views.append(flat[pos:pos + n])
            pos += n
        ex(views)
        want = expected(world, spec, mode, op, seed=3)
        ok2 = all(np.array_equal(v.numpy(), w.reshape(-1)) for v, w in zip(views, want))
        q.put((rank, ok and ok2))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,op", [("allgather", "avg"), ("two_round", "avg"), ("two_round", "sum")])
def test_gloo_world_size_2(mode, op):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, mode, op, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}


@pytest.mark.parametrize("nranks", [2, 4])
def test_model_parallel_fc_orchestration(nranks):
    """ModelParallelFC's gather / compressed-sum plumbing on CPU (test codec)."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    rng = np.random.default_rng(7)
    x = torch.from_numpy(rng.normal(0, 0.02, size=(16, 64)).astype(np.float32))
    w = torch.from_numpy(rng.normal(0, 0.02, size=(64, 32)).astype(np.float32))
    dy = torch.from_numpy(rng.normal(0, 1e-3, size=(16, 32)).astype(np.float32))
    k = 32 // nranks

    def body(rank, comm):
        fc = A.ModelParallelFC(w[:, rank * k:(rank + 1) * k].contiguous(), spec, comm=comm, codec=NumpyCodec(spec))
        y = fc.forward(x)
        dx, _ = fc.backward(dy)
        return y.numpy(), dx.numpy(), (x @ fc.w).numpy(), (dy[:, rank * k:(rank + 1) * k] @ fc.w.t()).numpy()

    res = run_virtual_ranks(nranks, body)
    y_want = np.concatenate([O.roundtrip(res[r][2], "dynamic-tree", "absmax") for r in range(nranks)], axis=1)
    dx_want = O.exchange_allgather([[res[r][3]] for r in range(nranks)], "dynamic-tree", "absmax", op="sum")[0]
    for r in range(nranks):
        assert np.array_equal(res[r][0], y_want)
        assert np.array_equal(res[r][1], dx_want)


# ---------------------------------------------------------------------------
# the DDP comm hook with a real DistributedDataParallel model (gloo, 2 ranks)


def _ddp_model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(20, 30), torch.nn.ReLU(), torch.nn.Linear(30, 5))


def _ddp_inputs(rank):
    g = torch.Generator().manual_seed(100 + rank)
    return torch.randn(8, 20, generator=g), torch.randn(8, 5, generator=g)


def _local_grads(rank):
    m = _ddp_model()
    x, y = _ddp_inputs(rank)
    torch.nn.functional.mse_loss(m(x), y).backward()
    return [p.grad.numpy().copy() for p in m.parameters()]


def _ddp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = SPECS[0]
        model = torch.nn.parallel.DistributedDataParallel(_ddp_model())
        model.register_comm_hook(A.DDPHookState(spec, codec=NumpyCodec(spec), check="sync"), A.a8_comm_hook)
        x, y = _ddp_inputs(rank)
        torch.nn.functional.mse_loss(model(x), y).backward()
        per_rank = [_local_grads(r) for r in range(world)]
        ok = True
        for i, p in enumerate(model.parameters()):
            want = O.exchange_allgather([[per_rank[r][i]] for r in range(world)], spec.kind.value,
                                        spec.normalization.value, spec.decades, "avg")[0]
            ok &= bool(np.array_equal(p.grad.numpy(), want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_gloo_world_size_2():
    """register_comm_hook(DDPHookState, a8_comm_hook) on a real DDP model:
    every parameter's gradient is the 8-bit all-gather average of the ranks'
    local gradients (per-parameter scales), bit-exact against the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ddp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}


@pytest.mark.parametrize("nranks", [2, 4])
def test_pipelined_two_round_orchestration(nranks):
    """Round-2 all-gather in K > 1 blocks (test codec, CPU): bit-exact with the
    unchunked two_round oracle."""
    spec = SPECS[0]

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode="two_round", op="avg", check="sync", codec=NumpyCodec(spec), comm=comm,
                                chunk_elems=256)
        ts = [torch.from_numpy(g) for g in grads_for(rank)]
        ex(ts)
        return [t.numpy().copy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    want = expected(nranks, spec, "two_round", "avg")
    for r in range(nranks):
        for a, b in zip(res[r], want):
            assert np.array_equal(a, b), r


@pytest.mark.parametrize("nranks", [1, 2, 4])
@pytest.mark.parametrize("chunk", [8 << 20, 256])
def test_local_fp32_orchestration(nranks, chunk):
    """local_fp32: each rank's own term is its float32
    gradient; every other rank's is the round trip of its codes."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")

    def body(rank, comm):
        ex = A.GradientExchange(spec, check="sync", codec=NumpyCodec(spec), comm=comm, local_fp32=True,
                                chunk_elems=chunk)
        ts = [torch.from_numpy(g) for g in grads_for(rank, seed=3)]
        ex(ts)
        return [t.numpy().copy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    g = [grads_for(r, seed=3) for r in range(nranks)]
    for r in range(nranks):
        want = O.exchange_allgather_local(g, r, "dynamic-tree", "absmax")
        for a, b in zip(res[r], want):
            assert np.array_equal(a, b), (r, nranks)
    if nranks == 1:
        for a, b in zip(res[0], g[0]):
            assert np.array_equal(a, b)  # N = 1: the gradient itself


def test_local_fp32_needs_allgather():
    with pytest.raises(A.UsageError):
        A.GradientExchange(A.DataTypeSpec("linear", "absmax"), mode="two_round", local_fp32=True)


# ---------------------------------------------------------------------------
# the 1-bit error-feedback exchange (GradientExchange("onebit"))

ONEBIT_SIZES = [(40, 30), (1,), (17,), (0,), (300,), (4, 4, 4), (5000,)]


def _onebit_grads(rank, step):
    rng = np.random.default_rng(500 + 31 * rank + step)
    return [rng.normal(0, 1e-2, size=s).astype(np.float32) for s in ONEBIT_SIZES]


@pytest.mark.parametrize("nranks", [1, 2, 4])
def test_onebit_exchange_chained_steps_match_oracle(nranks):
    """5 chained steps: per-rank residuals carried on each rank, bits +
    levels all-gathered, rank-ordered float32 average -- bit-exact against
    oracle.exchange_onebit (codecs.py:306-348 per rank)."""
    steps = 5

    def body(rank, comm):
        ex = A.GradientExchange("onebit", check="sync", codec=NumpyOneBitCodec(), comm=comm)
        outs = []
        for k in range(steps):
            ts = [torch.from_numpy(g) for g in _onebit_grads(rank, k)]
            ex(ts)
            outs.append([t.numpy().copy() for t in ts])
        return outs

    res = run_virtual_ranks(nranks, body)
    resid = [[np.zeros(int(np.prod(s))) .reshape(s) for s in ONEBIT_SIZES] for _ in range(nranks)]
    for k in range(steps):
        want = O.exchange_onebit([_onebit_grads(r, k) for r in range(nranks)], resid)
        for r in range(nranks):
            for a, b in zip(res[r][k], want):
                assert a.tobytes() == b.astype(np.float32).tobytes(), (r, k)


def test_onebit_exchange_nonfinite_raises_everywhere_and_keeps_residuals():
    def body(rank, comm):
        ex = A.GradientExchange("onebit", check="sync", codec=NumpyOneBitCodec(), comm=comm)
        ex([torch.from_numpy(g) for g in _onebit_grads(rank, 0)])
        before = {k: v.clone() for k, v in ex.residuals.items()}
        ts = [torch.from_numpy(g) for g in _onebit_grads(rank, 1)]
        if rank == 1:
            ts[6][3] = float("inf")
        try:
            ex(ts)
            return "ok", None
        except A.InputError:
            k6 = (6, ts[6].numel())  # the non-finite tensor's own residual is untouched (codecs.py:317-318)
            return "raised", torch.equal(before[k6], ex.residuals[k6])

    res = run_virtual_ranks(2, body)
    assert [r[0] for r in res] == ["raised", "raised"]
    assert res[1][1] is True


def test_onebit_exchange_rejects_unsupported():
    with pytest.raises(A.UsageError):
        A.GradientExchange("onebit", mode="two_round")
    with pytest.raises(A.UsageError):
        A.GradientExchange("onebit", graph=True)


def _ddp_onebit_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = torch.nn.parallel.DistributedDataParallel(_ddp_model())
        model.register_comm_hook(A.DDPHookState("onebit", codec=NumpyOneBitCodec(), check="sync"), A.a8_comm_hook)
        x, y = _ddp_inputs(rank)
        torch.nn.functional.mse_loss(model(x), y).backward()
        per_rank = [_local_grads(r) for r in range(world)]
        resid = [[np.zeros(g.shape) for g in per_rank[r]] for r in range(world)]
        ok = True
        for i, p in enumerate(model.parameters()):
            want = O.exchange_onebit([[per_rank[r][i]] for r in range(world)], [[resid[r][i]] for r in range(world)])[0]
            ok &= bool(np.array_equal(p.grad.numpy(), want))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_ddp_comm_hook_onebit_gloo_world_size_2():
    """DDPHookState("onebit"): a real DDP model's gradients are the 1-bit
    exchange average (one residual per parameter), bit-exact vs the oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ddp_onebit_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=5) for _ in range(2))
    assert results == {0: True, 1: True}


def test_amax_validation():
    """Producer maxima (GradientExchange(...)(..., amax=)): absmax specs only,
    one float32 per tensor on the tensors' device, CUDA only -- all checked
    before any codec work."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync", codec=NumpyCodec(spec))
    ts = [torch.zeros(10), torch.zeros(3)]
    with pytest.raises(A.UsageError, match="CUDA"):
        ex(ts, amax=torch.zeros(2))
    with pytest.raises(A.UsageError, match="2 maxima"):
        ex(ts, amax=torch.zeros(3))
    with pytest.raises(A.UsageError, match="2 maxima"):
        ex(ts, amax=torch.zeros(2, dtype=torch.float64))
    fixed = A.DataTypeSpec("mantissa", "none")
    with pytest.raises(A.UsageError, match="absmax"):
        A.GradientExchange(fixed, check="sync", codec=NumpyCodec(fixed))(ts, amax=torch.zeros(2))
    with pytest.raises(A.ConfigError):
        A.ModelParallelFC(torch.zeros(4, 2), spec, activation="gelu")
