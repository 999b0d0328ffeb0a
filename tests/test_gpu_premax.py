"""GPU parity of the producer-fused max (a8_produce_absmax) and the one-pass
encode that uses it (a8_encode_premax), SURVEY 8(f) row 4.

Bar: the producer's outputs equal the torch/NumPy expression of the
reference producer bit for bit (mlp.py:205-207 relu + mask; the float32
pre-scale), its maxima equal max|y| bit for bit, and every encode or
exchange given those maxima is bit-identical to the same call without them
(which the rest of the suite pins to the reference).  Wrong maxima must
raise, never read out of bounds.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu

SPEC = A.DataTypeSpec("dynamic-tree", "absmax")
SIZES = [0, 1, 3, 4095, 4096, 4097, 12289, 70001, 1 << 20, 3_000_001]


def grads(sizes, seed=0, sigma=1e-3):
    return [torch.from_numpy(O.sample_normal(n, seed + i, 0.0, sigma)) for i, n in enumerate(sizes)]


def absmax_bits(t):
    return int(t.abs().max().view(torch.int32)) if t.numel() else 0


def test_scale_absmax_matches_torch(cuda):
    xs = [g.to(cuda) for g in grads(SIZES)]
    xs[5][7] = -3.5  # the max on a negative element
    for alpha in (1.0, 0.125, 1.0 / 3.0):
        ts = [x.clone() for x in xs]
        m = A.scale_absmax_(ts, alpha)
        for x, t, mi in zip(xs, ts, m.view(torch.int32).cpu()):
            want = x * torch.tensor(alpha, dtype=torch.float32, device=cuda)
            assert torch.equal(t.view(torch.int32), want.view(torch.int32))
            assert int(mi) == absmax_bits(want)


def test_scale_absmax_unaligned_views(cuda):
    base = grads([1 << 16])[0].to(cuda)
    views = [base[1:40001], base[3:5], base[5:5 + 8192 + 3]]  # not 16-byte aligned
    ref = [v.clone() for v in views]
    m = A.scale_absmax_([v.contiguous() for v in views], 1.0)
    for r, mi in zip(ref, m.view(torch.int32).cpu()):
        assert int(mi) == absmax_bits(r)


@pytest.mark.parametrize("masked", [False, True])
def test_relu_absmax_matches_reference_producer(cuda, masked):
    rng = np.random.default_rng(5)
    z = rng.normal(0, 1, (257, 1031)).astype(np.float32)
    z[0, :4] = [-0.0, np.nan, 0.0, -np.inf]
    mask = ((rng.random(z.shape) >= 0.5) / 0.5).astype(np.float32) if masked else None
    h, m = A.relu_absmax(torch.from_numpy(z).to(cuda), None if mask is None else torch.from_numpy(mask).to(cuda))
    want = np.maximum(z, np.float32(0.0))  # mlp.py:205
    if masked:
        want = want * mask  # mlp.py:207 (float32 here)
    got = h.cpu().numpy()
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    if not masked:  # np.maximum keeps the NaN's bits; a float multiply makes its own NaN
        assert got.tobytes() == want.tobytes()
    assert got[~nan].tobytes() == want[~nan].tobytes()
    assert np.isnan(m.cpu().numpy()[0])  # the max of a tensor holding NaN is NaN (encode then raises)
    z[0, 1] = 0.0
    h, m = A.relu_absmax(torch.from_numpy(z).to(cuda), None if mask is None else torch.from_numpy(mask).to(cuda))
    want = np.maximum(z, np.float32(0.0)) * (mask if masked else np.float32(1))
    assert h.cpu().numpy().tobytes() == want.astype(np.float32).tobytes()
    assert int(m.view(torch.int32).cpu()[0]) == int(np.abs(want).max().view(np.int32))


def test_encode_buffer_premax_identical(cuda):
    cb = A.build_codebook(SPEC)
    for n in SIZES[1:]:
        x = grads([n], seed=n)[0].to(cuda)
        m = A.scale_absmax_([x], 1.0)
        a, b = A.encode_buffer(x, cb), A.encode_buffer(x, cb, amax=m)
        assert a.scale == b.scale
        assert torch.equal(a.codes_device, b.codes_device)


def test_exchange_premax_identical_c3_shapes(cuda):
    """The bench's config-3 tensors (AlexNet shapes), producer pre-scale 1/2
    then the exchange with its maxima, against the two-pass exchange."""
    import bench

    host = bench.alexnet_grads(0)
    for mode in ("allgather", "two_round"):
        a = [torch.from_numpy(g).to(cuda).reshape(-1) for g in host]
        b = [t.clone() for t in a]
        for t in a:
            t.mul_(0.5)
        A.GradientExchange(SPEC, mode=mode, check="sync")(a)
        ex = A.GradientExchange(SPEC, mode=mode, check="sync")
        for step in range(2):  # the second call replays the recorded step
            bb = [t.clone() for t in b]
            m = A.scale_absmax_(bb, 0.5)
            ex(bb, amax=m)
            for x, y in zip(a, bb):
                assert torch.equal(x.view(torch.int32), y.view(torch.int32)), mode


def test_exchange_premax_graph_mode(cuda):
    xs = [g.to(cuda) for g in grads([70001, 4096, 9, 1 << 18])]
    want = [x.clone() for x in xs]
    A.GradientExchange(SPEC, check="sync")(want)
    ex = A.GradientExchange(SPEC, check="sync", graph=True)
    m = torch.empty(len(xs), dtype=torch.float32, device=cuda)
    bufs = [x.clone() for x in xs]
    for _ in range(3):
        for b, x in zip(bufs, xs):
            b.copy_(x)
        m.copy_(A.scale_absmax_(bufs, 1.0))
        ex(bufs, amax=m)
        for b, w in zip(bufs, want):
            assert torch.equal(b, w)


@pytest.mark.parametrize("n", [9, 4096, 70001, 3_000_001, 9_000_001])
def test_wrong_amax_raises(cuda, n):
    """Smaller (elements above the table: clamped, no stray reads), larger
    and off-by-one-ulp maxima are all reported."""
    cb = A.build_codebook(SPEC)
    x = grads([n], seed=3)[0].to(cuda)
    true = A.scale_absmax_([x], 1.0)
    for bad in (true * 0.25, true * 2.0, (true.view(torch.int32) - 1).view(torch.float32)):
        with pytest.raises(A.UsageError):
            A.encode_buffer(x, cb, amax=bad.clone())
    ex = A.GradientExchange(SPEC, check="sync")
    with pytest.raises(A.UsageError):
        ex([x.clone()], amax=true * 0.5)
    # the exchange still works afterwards
    y = x.clone()
    ex([y], amax=true)
    z = x.clone()
    A.GradientExchange(SPEC, check="sync")([z])
    assert torch.equal(y, z)


def test_premax_nonfinite_raises_inputerror(cuda):
    x = grads([100_000])[0].to(cuda)
    x[777] = float("nan")
    m = A.scale_absmax_([x], 1.0)
    assert torch.isnan(m).all()
    with pytest.raises(A.InputError):
        A.GradientExchange(SPEC, check="sync")([x], amax=m)


def test_amax_usage_errors(cuda):
    x = grads([1000])[0].to(cuda)
    with pytest.raises(A.UsageError):
        A.GradientExchange(A.DataTypeSpec("mantissa", "none"), check="sync")([x], amax=torch.ones(1, device=cuda))
    with pytest.raises(A.UsageError):
        A.GradientExchange(SPEC, check="sync")([x], amax=torch.ones(2, device=cuda))
    with pytest.raises(A.UsageError):
        A.encode_buffer(x, A.build_codebook(SPEC), amax=torch.ones(1, dtype=torch.float64, device=cuda))


def test_model_parallel_relu_ships_relu_activation(cuda):
    """ModelParallelFC(activation="relu") at world size 1: the gathered
    activation is the round trip of h = relu(x @ W) * mask, and backward
    applies the gate (mlp.py:205-209, 250-253)."""
    g = torch.Generator().manual_seed(0)
    w = (torch.randn(64, 48, generator=g) * 0.1).to(cuda)
    x = torch.randn(16, 64, generator=g).to(cuda)
    mask = ((torch.rand(16, 48, generator=g) >= 0.5).float() / 0.5).to(cuda)
    fc = A.ModelParallelFC(w, SPEC, activation="relu")
    y = fc.forward(x, mask)
    h = torch.from_numpy(np.maximum((x @ w).cpu().numpy(), np.float32(0)) * mask.cpu().numpy())
    want = O.roundtrip(h.numpy().reshape(-1), "dynamic-tree", "absmax").reshape(h.shape)
    assert y.cpu().numpy().tobytes() == want.tobytes()
    dy = torch.randn(16, 48, generator=g).to(cuda)
    dx, dw = fc.backward(dy)
    dz = dy * ((x @ w) > 0).float() * mask
    assert torch.allclose(dw, x.t() @ dz, rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("mode", ["allgather", "two_round"])
def test_peer_exchange_premax_matches_oracle(cuda, mode):
    """PeerExchange (virtual ranks on one GPU) with every rank's maxima from
    its producer pass: bit-exact against the composed oracle."""
    from helpers import run_virtual_peers

    sizes = [5, 4096, 70001, 300_000]

    def per(rank, step):
        return [O.sample_normal(n, 100 * rank + 10 * step + i, 0.0, 1e-3) for i, n in enumerate(sizes)]

    def body(rank, peers):
        ex = A.PeerExchange(SPEC, peers, mode=mode, check="sync")
        res = []
        for step in range(2):
            ts = [torch.from_numpy(g).to(cuda) for g in per(rank, step)]
            ex(ts, amax=A.scale_absmax_(ts, 1.0))
            res.append([t.cpu().numpy() for t in ts])
        return res

    res = run_virtual_peers(3, body)
    for step in range(2):
        ins = [per(r, step) for r in range(3)]
        want = (O.exchange_allgather(ins, "dynamic-tree", "absmax") if mode == "allgather"
                else O.exchange_two_round(ins, "dynamic-tree", "absmax"))
        for r in range(3):
            for a, b in zip(res[r][step], want):
                assert a.tobytes() == b.astype(np.float32).tobytes(), (r, step)


def test_premax_many_segments(cuda):
    """More tensors than the launch-inline plan (32) and the shared-memory
    maxima (64): the plan and the maxima go through global memory."""
    sizes = [(7 * i * i + 3) % 20000 + 1 for i in range(70)] + [300_000, 4096 * 3]
    xs = [g.to(cuda) for g in grads(sizes, seed=11)]
    want = [x.clone() for x in xs]
    A.GradientExchange(SPEC, check="sync")(want)
    got = [x.clone() for x in xs]
    A.GradientExchange(SPEC, check="sync")(got, amax=A.scale_absmax_(got, 1.0))
    for a, b in zip(got, want):
        assert torch.equal(a, b)
    bad = A.scale_absmax_(got, 1.0)
    bad[69] = bad[69] * 0.5
    with pytest.raises(A.UsageError):
        A.GradientExchange(SPEC, check="sync")([x.clone() for x in xs], amax=bad)
