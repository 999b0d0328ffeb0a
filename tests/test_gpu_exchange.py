"""GPU parity of the compressed exchange (allgather / two_round, avg / sum).

One GPU: N ranks are simulated as N threads (``ThreadComm``) that each drive
the real CUDA codec on the same device; the collectives are buffer copies.
The result must equal the composed oracle (oracle.exchange_*) -- bit-exact in
practice; the contract tolerance is 1e-6 relative in float32, written below.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O, run_virtual_ranks

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu

ALEXNET = [(64, 3, 11, 11), (64,), (192, 64, 5, 5), (192,), (384, 192, 3, 3), (384,),
           (256, 384, 3, 3), (256,), (256, 256, 3, 3), (256,), (4096, 9216), (4096,),
           (4096, 4096), (4096,), (1000, 4096), (1000,)]
SMALL = [(40, 30), (1,), (17,), (0,), (300,), (4, 4, 4), (5000,), (70000,)]
RTOL = 1e-6  # north-star tolerance for averaged outputs (float32)


def grads(rank, sizes, seed=0, sigma=1e-2):
    rng = np.random.default_rng(seed * 1000 + rank)
    return [rng.normal(0.0, sigma, size=s).astype(np.float32) for s in sizes]


def close(a, b):
    a64, b64 = a.astype(np.float64), b.astype(np.float64)
    return bool(np.all(np.abs(a64 - b64) <= RTOL * np.abs(b64) + 1e-45))


def run(nranks, sizes, spec, mode, op, cuda, seed=0):
    def body(rank, comm):
        ex = A.GradientExchange(spec, mode=mode, op=op, check="sync", comm=comm)
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, sizes, seed)]
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    g = [grads(r, sizes, seed) for r in range(nranks)]
    fn = O.exchange_allgather if mode == "allgather" else O.exchange_two_round
    want = fn(g, spec.kind.value, spec.normalization.value, spec.decades, op)
    return res, want


def test_world_size_one_is_roundtrip(cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync")
    gs = grads(0, SMALL + ALEXNET[:4])
    ts = [torch.from_numpy(g).to(cuda) for g in gs]
    ex(ts)
    for t, g in zip(ts, gs):
        assert t.cpu().numpy().tobytes() == O.roundtrip(g, "dynamic-tree", "absmax").tobytes()


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("mode", ["allgather", "two_round"])
@pytest.mark.parametrize("op", ["avg", "sum"])
def test_virtual_ranks_match_oracle(nranks, mode, op, cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    res, want = run(nranks, SMALL, spec, mode, op, cuda)
    for r in range(nranks):
        for a, b in zip(res[r], want):
            assert a.shape == b.shape
            assert close(a, b), (r, mode, op)
            assert a.tobytes() == b.tobytes(), (r, mode, op)  # bit-exact in practice


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("chunk", [4096, 20000])
def test_pipelined_allgather_chunks(nranks, chunk, cuda):
    """allgather with K > 1 chunk-blocks (pieces split at chunk boundaries)."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode="allgather", check="sync", comm=comm, chunk_elems=chunk)
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, SMALL, 7)]
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    want = O.exchange_allgather([grads(r, SMALL, 7) for r in range(nranks)], "dynamic-tree", "absmax")
    for r in range(nranks):
        for a, b in zip(res[r], want):
            assert a.tobytes() == b.tobytes(), (r, nranks, chunk)


@pytest.mark.parametrize("spec", [A.DataTypeSpec("linear", "absmax"), A.DataTypeSpec("mantissa", "none"),
                                  A.DataTypeSpec("static-tree", "decade", -2)], ids=lambda s: s.label())
def test_other_specs_three_ranks(spec, cuda):
    for mode in ("allgather", "two_round"):
        res, want = run(3, SMALL, spec, mode, "avg", cuda, seed=4)
        for r in range(3):
            for a, b in zip(res[r], want):
                assert a.tobytes() == b.tobytes(), (spec.label(), mode, r)


def test_alexnet_shapes_two_ranks(cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    for mode in ("allgather", "two_round"):
        res, want = run(2, ALEXNET, spec, mode, "avg", cuda, seed=9)
        for r in range(2):
            for a, b in zip(res[r], want):
                assert a.tobytes() == b.tobytes(), (mode, r)


@pytest.mark.parametrize("mode", ["allgather", "two_round"])
def test_non_finite_raises_on_every_rank(mode, cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode=mode, check="sync", comm=comm)
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, SMALL)]
        if rank == 2:
            ts[6][123] = float("inf")
        try:
            ex(ts)
        except A.InputError:
            return "raised"
        return "ok"

    assert run_virtual_ranks(4, body) == ["raised"] * 4


def test_many_segments_use_device_plan(cuda):
    """> 48 tensors: descriptors go through the workspace instead of the launch."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    sizes = [(int(n),) for n in np.random.default_rng(2).integers(1, 3000, size=130)]
    res, want = run(2, sizes, spec, "allgather", "avg", cuda, seed=5)
    for r in range(2):
        for a, b in zip(res[r], want):
            assert a.tobytes() == b.tobytes()


def test_model_parallel_quantizer_seam(cuda):
    """mlp.py:167-175 seam on the GPU: quantize(x) == roundtrip, stats recorded."""
    spec = A.default_hook_spec("dynamic-tree", "model-parallel")
    stats = A.HookStats()
    qz = A.make_quantizer(spec, stats, "forward")
    x = torch.relu(torch.randn(128, 512, device=cuda))
    y = qz(x, 1)
    assert torch.equal(y, A.roundtrip(x, spec))
    s = stats.summary()["forward"][0]
    assert s[0] > 0 and 0 < s[1] < 5


def test_graph_mode_replays_match_roundtrip(cuda):
    """graph=True: first call eager + capture, later calls replay; every call
    equals the per-tensor round trip of that call's data (buffers reused)."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync", graph=True)
    sizes = SMALL + ALEXNET[:6]
    ins = [torch.empty(s, device=cuda) for s in sizes]
    outs = [torch.empty(s, device=cuda) for s in sizes]
    for step in range(4):
        gs = grads(0, sizes, seed=10 + step)
        for t, g in zip(ins, gs):
            t.copy_(torch.from_numpy(g))
        ex(ins, out=outs)
        for o, g in zip(outs, gs):
            assert o.cpu().numpy().tobytes() == O.roundtrip(g, "dynamic-tree", "absmax").tobytes(), step
    assert len(ex._graphs) == 1
    # other output buffers -> a second graph
    outs2 = [torch.empty_like(o) for o in outs]
    ex(ins, out=outs2)
    ex(ins, out=outs2)
    assert len(ex._graphs) == 2
    for a, b in zip(outs, outs2):
        assert torch.equal(a, b)


def test_graph_mode_reports_non_finite(cuda):
    spec = A.DataTypeSpec("linear", "absmax")
    ex = A.GradientExchange(spec, check="sync", graph=True)
    ts = [torch.randn(1000, device=cuda), torch.randn(77, device=cuda)]
    outs = [torch.empty_like(t) for t in ts]
    ex(ts, out=outs)
    ex(ts, out=outs)  # replay
    ts[1][5] = float("inf")
    with pytest.raises(A.InputError):
        ex(ts, out=outs)
    ts[1][5] = 0.0
    ex(ts, out=outs)  # clean again
    assert torch.isfinite(outs[1]).all()


def test_graph_mode_deferred_reports_every_bad_replay(cuda):
    """replays share one host word; with check='deferred' a bad
    replay followed by a clean one before any check must still raise."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, graph=True)  # check="deferred"
    ts = [torch.randn(3000, device=cuda), torch.randn(77, device=cuda)]
    outs = [torch.empty_like(t) for t in ts]
    ex(ts, out=outs)
    ex(ts, out=outs)
    ex.synchronize()
    ts[0][7] = float("nan")
    ex(ts, out=outs)  # bad replay, not checked yet
    ts[0][7] = 1.0
    with pytest.raises(A.InputError):
        ex(ts, out=outs)  # clean replay: overwrites nothing (the word counts); may see the bad one
        ex.synchronize()
    ex(ts, out=outs)
    ex.synchronize()  # reported once, clean afterwards


def test_graph_mode_survives_workspace_growth(cuda):
    """a call with more tensors but no more bytes must not leave a
    captured graph pointing at a freed workspace."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync", graph=True)
    few = [(20000,), (5000,)]
    many = [(700,)] * 30
    fi = [torch.from_numpy(g).to(cuda) for g in grads(0, few, seed=1)]
    fo = [torch.empty_like(t) for t in fi]
    mi = [torch.from_numpy(g).to(cuda) for g in grads(0, many, seed=2)]
    mo = [torch.empty_like(t) for t in mi]
    for _ in range(3):
        ex(fi, out=fo)
        ex(mi, out=mo)
    # a 40-segment eager call on the side stream grows nothing the graphs use
    big = [torch.from_numpy(g).to(cuda) for g in grads(0, [(300,)] * 40, seed=3)]
    ex(big)
    for _ in range(2):
        ex(fi, out=fo)
        ex(mi, out=mo)
    for t, o in zip(fi + mi, fo + mo):
        assert o.cpu().numpy().tobytes() == O.roundtrip(t.cpu().numpy(), "dynamic-tree", "absmax").tobytes()


def test_exchange_validates_out(cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync")
    ts = [torch.randn(100, device=cuda)]
    for bad in ([torch.empty(100, device=cuda, dtype=torch.float16)], [torch.empty(99, device=cuda)],
                [torch.empty(200, device=cuda)[::2]], []):
        with pytest.raises(A.UsageError):
            ex(ts, out=bad)


def test_make_quantizer_f64_non_finite_raises(cuda):
    """the non-fused (float64) quantizer path raises InputError like mlp.py:171."""
    qz = A.make_quantizer(A.DataTypeSpec("dynamic-tree", "absmax"))
    x = torch.randn(64, 10, dtype=torch.float64, device=cuda)
    qz(x, 0)
    x[3, 4] = float("inf")
    with pytest.raises(A.InputError):
        qz(x, 0)


def test_graph_mode_many_tensors_runs_eagerly(cuda):
    """> 32 tensors: the launch plan goes through device memory, no capture."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="sync", graph=True)
    sizes = [(int(n),) for n in np.random.default_rng(9).integers(1, 500, size=40)]
    gs = grads(0, sizes, seed=3)
    ts = [torch.from_numpy(g).to(cuda) for g in gs]
    ex(ts)
    assert not ex._graphs
    for t, g in zip(ts, gs):
        assert t.cpu().numpy().tobytes() == O.roundtrip(g, "dynamic-tree", "absmax").tobytes()


def test_deferred_checks_every_call(cuda):
    """check="deferred": a non-finite input in call k is reported even when
    later calls were issued before it was checked (status ring, one
    host-mapped word per call)."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    ex = A.GradientExchange(spec, check="deferred")
    good = [torch.randn(5000, device=cuda), torch.randn(33, device=cuda)]
    bad = [good[0].clone(), good[1].clone()]
    bad[0][123] = float("nan")
    outs = [torch.empty_like(t) for t in good]
    ex(good, out=outs)
    ex(bad, out=outs)
    with pytest.raises(A.InputError, match="call 1"):
        for _ in range(5):  # raised by a later call's poll, or at the latest by synchronize
            ex(good, out=outs)
        ex.synchronize()
    ex(good, out=outs)
    ex.synchronize()  # clean again


def test_functional_exchange_world_size_one(cuda):
    """exchange(tensors, spec): the one-shot form (check="sync")."""
    spec = A.DataTypeSpec("linear", "absmax")
    gs = grads(0, SMALL, seed=21)
    ts = [torch.from_numpy(g).to(cuda) for g in gs]
    out = A.exchange(ts, spec)
    assert out is not None
    for t, g in zip(ts, gs):
        assert t.cpu().numpy().tobytes() == O.roundtrip(g, "linear", "absmax").tobytes()


@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("chunk", [4096, 50000])
def test_pipelined_two_round_chunks(nranks, chunk, cuda):
    """two_round with the round-2 all-gather split into K > 1 blocks: same
    pieces and scales as K = 1, so bit-exact against the unchunked oracle."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")

    def body(rank, comm):
        ex = A.GradientExchange(spec, mode="two_round", check="sync", comm=comm, chunk_elems=chunk)
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, SMALL + ALEXNET[:2], 9)]
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    want = O.exchange_two_round([grads(r, SMALL + ALEXNET[:2], 9) for r in range(nranks)], "dynamic-tree", "absmax")
    for r in range(nranks):
        for a, b in zip(res[r], want):
            assert a.tobytes() == b.tobytes(), (r, nranks, chunk)


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
@pytest.mark.parametrize("chunk", [8 << 20, 20000])
def test_local_fp32_matches_oracle(nranks, chunk, cuda):
    """local_fp32 through a8_decode_local, in place, bit-exact
    against the per-rank oracle; ranks hold different results."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    sizes = SMALL + ALEXNET[:4]

    def body(rank, comm):
        ex = A.GradientExchange(spec, check="sync", comm=comm, local_fp32=True, chunk_elems=chunk)
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, sizes, 11)]
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    g = [grads(r, sizes, 11) for r in range(nranks)]
    for r in range(nranks):
        want = O.exchange_allgather_local(g, r, "dynamic-tree", "absmax")
        for a, b in zip(res[r], want):
            assert a.tobytes() == b.tobytes(), (r, nranks, chunk)


def test_local_fp32_unaligned_pieces(cuda):
    """Outputs and local inputs at offsets that are not 16-byte aligned take
    the scalar path of the kernel."""
    spec = A.DataTypeSpec("linear", "absmax")

    def body(rank, comm):
        base = torch.from_numpy(np.concatenate([np.zeros(1, np.float32)] + grads(rank, [(9001,), (4099,)], 12))).to(cuda)
        ts = [base[1:9002], base[9002:]]
        ex = A.GradientExchange(spec, check="sync", comm=comm, local_fp32=True)
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(2, body)
    g = [grads(r, [(9001,), (4099,)], 12) for r in range(2)]
    for r in range(2):
        want = O.exchange_allgather_local(g, r, "linear", "absmax")
        for a, b in zip(res[r], want):
            assert a.tobytes() == b.tobytes(), r


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_onebit_exchange_virtual_ranks_match_oracle(cuda, nranks):
    """GradientExchange("onebit") with the CUDA kernels: 5 chained steps, one
    device residual per tensor and rank, bit-exact against
    oracle.exchange_onebit (per-rank onebit_quantize, codecs.py:306-348;
    rank-ordered float32 average)."""
    sizes = SMALL + ALEXNET[:4]
    steps = 5

    def g(rank, k):
        rng = np.random.default_rng(900 + 17 * rank + k)
        return [rng.normal(0, 1e-2, size=s).astype(np.float32) for s in sizes]

    def body(rank, comm):
        ex = A.GradientExchange("onebit", check="sync", comm=comm)
        outs = []
        for k in range(steps):
            ts = [torch.from_numpy(x).to(cuda) for x in g(rank, k)]
            ex(ts)
            outs.append([t.cpu().numpy() for t in ts])
        return outs

    res = run_virtual_ranks(nranks, body)
    resid = [[np.zeros(s) for s in sizes] for _ in range(nranks)]
    for k in range(steps):
        want = O.exchange_onebit([g(r, k) for r in range(nranks)], resid)
        for r in range(nranks):
            for a, b in zip(res[r][k], want):
                assert a.tobytes() == b.astype(np.float32).tobytes(), (r, k)


def test_onebit_exchange_many_tensors_and_float64(cuda):
    """> 32 tensors (several reduce launches, one status OR) and float64
    gradients (the reference seam's dtype) at N = 1 == the chained 1-bit
    round trip of each tensor."""
    rng = np.random.default_rng(4)
    sizes = [int(v) for v in rng.integers(1, 3000, size=40)]
    ex = A.GradientExchange("onebit", check="sync")
    resid = [[np.zeros(n) for n in sizes]]
    for k in range(3):
        xs = [rng.normal(size=n) for n in sizes]
        ins = [torch.from_numpy(x).to(cuda) for x in xs]
        outs = [torch.empty(n, device=cuda) for n in sizes]
        ex(ins, out=outs)
        want = O.exchange_onebit([xs], resid)
        for o, w in zip(outs, want):
            assert o.cpu().numpy().tobytes() == w.astype(np.float32).tobytes(), k
    bad = [torch.from_numpy(rng.normal(size=n)).to(cuda) for n in sizes]
    bad[37][0] = float("nan")
    with pytest.raises(A.InputError):
        ex(bad, out=[torch.empty(n, device=cuda) for n in sizes])


@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["allgather", "two_round"])
@pytest.mark.parametrize("op", ["avg", "sum"])
def test_peer_exchange_matches_oracle(cuda, nranks, mode, op):
    """PeerExchange: the decode reads every rank's slab directly
    (a8_decode_peers over peer addresses; here virtual ranks on one GPU),
    3 calls (both double-buffer parities) bit-exact against the oracle."""
    from helpers import run_virtual_peers

    sizes = SMALL + ALEXNET[:5]

    def body(rank, peers):
        ex = A.PeerExchange(A.DataTypeSpec("dynamic-tree", "absmax"), peers, mode=mode, op=op, check="sync")
        res = []
        for step in range(3):
            ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, sizes, seed=step)]
            ex(ts)
            res.append([t.cpu().numpy() for t in ts])
        return res

    res = run_virtual_peers(nranks, body)
    for step in range(3):
        per = [grads(r, sizes, seed=step) for r in range(nranks)]
        want = (O.exchange_allgather(per, "dynamic-tree", "absmax", op=op) if mode == "allgather"
                else O.exchange_two_round(per, "dynamic-tree", "absmax", op=op))
        for r in range(nranks):
            for a, b in zip(res[r][step], want):
                assert a.tobytes() == b.astype(np.float32).tobytes(), (r, step)


def test_peer_exchange_nonfinite_raises_on_every_rank(cuda):
    from helpers import run_virtual_peers

    def body(rank, peers):
        ex = A.PeerExchange(A.DataTypeSpec("linear", "absmax"), peers, mode="two_round", check="sync")
        ts = [torch.from_numpy(g).to(cuda) for g in grads(rank, SMALL)]
        if rank == 2:
            ts[6][11] = float("inf")
        try:
            ex(ts)
        except A.InputError:
            return "raised"
        return "ok"

    from helpers import run_virtual_peers as rvp
    assert rvp(3, body) == ["raised"] * 3


@pytest.mark.parametrize("nranks", [2, 4])
@pytest.mark.parametrize("mode", ["allgather", "two_round"])
def test_recorded_step_replays_match_oracle(cuda, nranks, mode):
    """The eager step is recorded on its first call and replayed afterwards
    (_StepRecorder): 4 calls with new data in the same tensors, each
    bit-exact against the oracle; a non-finite input on one rank in a
    replayed call raises on every rank (the status word is re-pointed)."""
    sizes = SMALL + ALEXNET[:5]

    def body(rank, comm):
        ex = A.GradientExchange(A.DataTypeSpec("dynamic-tree", "absmax"), mode=mode, check="sync", comm=comm,
                                chunk_elems=1 << 16)
        ts = [torch.empty(s, device=cuda) for s in sizes]
        res = []
        for step in range(4):
            for t, g in zip(ts, grads(rank, sizes, seed=20 + step)):
                t.copy_(torch.from_numpy(g))
            ex(ts)
            res.append([t.cpu().numpy() for t in ts])
        assert len(ex._prepared) == 1
        for t, g in zip(ts, grads(rank, sizes, seed=99)):
            t.copy_(torch.from_numpy(g))
        if rank == nranks - 1:
            ts[6][3] = float("nan")
        try:
            ex(ts)
            res.append("ok")
        except A.InputError:
            res.append("raised")
        return res

    res = run_virtual_ranks(nranks, body)
    for step in range(4):
        per = [grads(r, sizes, seed=20 + step) for r in range(nranks)]
        want = (O.exchange_allgather(per, "dynamic-tree", "absmax") if mode == "allgather"
                else O.exchange_two_round(per, "dynamic-tree", "absmax"))
        for r in range(nranks):
            for a, b in zip(res[r][step], want):
                assert a.tobytes() == b.astype(np.float32).tobytes(), (r, step)
    assert [res[r][4] for r in range(nranks)] == ["raised"] * nranks


def test_recorded_steps_are_bounded(cuda):
    """Fresh tensors every call (new addresses): at most _PREPARED_MAX
    recordings are kept, and every call stays correct."""
    ex = A.GradientExchange(A.DataTypeSpec("dynamic-tree", "absmax"), check="sync")
    for step in range(A.GradientExchange._PREPARED_MAX + 5):
        gs = grads(0, SMALL, seed=step)
        ts = [torch.from_numpy(g).to(cuda) for g in gs]
        keep = [t.clone() for t in ts]  # hold the previous tensors so addresses differ
        ex(ts)
        for t, g in zip(ts, gs):
            assert t.cpu().numpy().tobytes() == O.roundtrip(g, "dynamic-tree", "absmax").tobytes(), step
        del keep
    assert len(ex._prepared) <= A.GradientExchange._PREPARED_MAX
