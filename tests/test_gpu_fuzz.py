"""Seeded random calls against the C oracle (oracle/approx8_oracle.c, the
restatement of codecs.py:244-288 pinned to the reference goldens).

Each case draws a spec (every kind / norm the reference allows, decades
-7..7), 1-32 tensors with sizes from 0 to a few million (log-uniform, so
every kernel path is hit: resident, ticket, single-chunk F segments, ragged
tails), magnitudes from subnormal to 1e30, several distributions, and
pointers that are not 16-byte aligned (views into a larger buffer).  The
N = 1 exchange (one encode launch for all tensors, one decode launch) must
reproduce the oracle's round trip of every tensor bit for bit, and
``encode_buffer`` its codes and scale; likewise the per-block codec, the
producer-fused maxima + one-pass encode, and N = 2..5 virtual-rank
exchanges.  Cases with a NaN / Inf planted in
one tensor must raise ``InputError`` and leave the codec usable.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu

SPECS = ["dynamic-tree/absmax", "linear/absmax", "dynamic-tree", "linear", "static-tree", "mantissa"] + [
    f"{k}/decade{d:+d}" for k in ("static-tree", "mantissa") for d in (-7, -3, 0, 2, 7)]


def _oracle_args(label):
    kind, _, norm = label.partition("/")
    if norm.startswith("decade"):
        return kind, "decade", int(norm[6:])
    return kind, norm or "none", 0


def _draw(rng, nseg, max_n):
    sizes = []
    for _ in range(nseg):
        r = rng.random()
        if r < 0.1:
            sizes.append(0)
        elif r < 0.3:
            sizes.append(int(rng.integers(1, 4097)))
        else:
            sizes.append(int(np.exp(rng.uniform(np.log(4096), np.log(max_n)))))
    host = []
    for n in sizes:
        mag = 10.0 ** rng.uniform(-30, 30) if rng.random() < 0.8 else float(rng.choice([1e-40, 1e-44, 3e38]))
        kind = rng.integers(0, 4)
        if kind == 0:
            x = rng.standard_normal(n) * mag
        elif kind == 1:
            x = rng.uniform(-mag, mag, n)
        elif kind == 2:  # heavy tails
            x = rng.standard_cauchy(n) * mag
        else:  # sparse, with exact zeros and repeated values
            x = np.where(rng.random(n) < 0.7, 0.0, np.round(rng.standard_normal(n) * 4) * mag)
        with np.errstate(over="ignore"):
            x = np.nan_to_num(x.astype(np.float32), nan=0.0, posinf=3e38, neginf=-3e38)
        host.append(x)
    return host


def _to_device(rng, host, dev):
    """Contiguous views at random element offsets (pointers not 16-byte aligned)."""
    out = []
    for h in host:
        off = int(rng.integers(0, 4))
        buf = torch.empty(h.size + off, dtype=torch.float32, device=dev)
        v = buf[off:off + h.size]
        v.copy_(torch.from_numpy(h))
        out.append(v)
    return out


@pytest.mark.parametrize("case", range(24))
def test_exchange_matches_oracle(cuda, case):
    rng = np.random.default_rng(9000 + case)
    label = SPECS[case % len(SPECS)]
    kind, norm, dec = _oracle_args(label)
    nseg = int(rng.integers(1, 33))
    host = _draw(rng, nseg, 3_000_000 if case % 3 else 12_000_000)
    grads = _to_device(rng, host, cuda)
    outs = [torch.full_like(g, float("nan")) for g in grads]
    A.GradientExchange(A.parse_spec(label), check="sync")(grads, out=outs)
    for i, (h, o) in enumerate(zip(host, outs)):
        c, s = O.c_encode(h, kind, norm, dec)
        want = O.c_decode(c, s, kind)
        assert o.cpu().numpy().tobytes() == want.tobytes(), (label, i, h.size)


@pytest.mark.parametrize("case", range(12))
def test_encode_buffer_matches_oracle(cuda, case):
    rng = np.random.default_rng(9500 + case)
    label = SPECS[(3 * case) % len(SPECS)]
    kind, norm, dec = _oracle_args(label)
    (h,) = _draw(rng, 1, 10_000_000)
    (x,) = _to_device(rng, [h], cuda)
    q = A.encode_buffer(x, A.build_codebook(A.parse_spec(label)))
    c, s = O.c_encode(h, kind, norm, dec)
    codes = q.codes.cpu().numpy() if hasattr(q.codes, "cpu") else np.asarray(q.codes)
    assert codes.tobytes() == c.tobytes(), label
    assert np.float32(q.scale) == np.float32(s)


@pytest.mark.parametrize("case", range(8))
def test_non_finite_anywhere_raises(cuda, case):
    rng = np.random.default_rng(9900 + case)
    label = ["dynamic-tree/absmax", "linear/absmax", "mantissa/decade+1", "static-tree"][case % 4]
    host = _draw(rng, int(rng.integers(2, 20)), 6_000_000)
    host = [h if h.size else np.ones(5, np.float32) for h in host]
    grads = _to_device(rng, host, cuda)
    outs = [torch.empty_like(g) for g in grads]
    ex = A.GradientExchange(A.parse_spec(label), check="sync")
    t = int(rng.integers(0, len(grads)))
    j = int(rng.integers(0, grads[t].numel()))
    grads[t][j] = [float("nan"), float("inf"), -float("inf")][case % 3]
    with pytest.raises(A.InputError):
        ex(grads, out=outs)
    grads[t][j] = 0.0
    host[t][j] = 0.0
    ex(grads, out=outs)
    kind, norm, dec = _oracle_args(label)
    for h, o in zip(host, outs):
        c, s = O.c_encode(h, kind, norm, dec)
        assert o.cpu().numpy().tobytes() == O.c_decode(c, s, kind).tobytes()


@pytest.mark.parametrize("case", range(8))
def test_virtual_ranks_match_oracle(cuda, case):
    """N = 2..5 ranks (threads driving the real codec, collectives as buffer
    copies), random specs and tensor lists, both modes, avg and sum, against
    the composed oracle (oracle.exchange_allgather / exchange_two_round)."""
    from helpers import run_virtual_ranks

    rng = np.random.default_rng(9700 + case)
    label = SPECS[(5 * case) % len(SPECS)]
    kind, norm, dec = _oracle_args(label)
    nranks = int(rng.integers(2, 6))
    mode = ("allgather", "two_round")[case % 2]
    op = ("avg", "sum")[(case // 2) % 2]
    nseg = int(rng.integers(1, 12))
    per_rank = [_draw(np.random.default_rng(9800 + 10 * case + r), nseg, 400_000) for r in range(nranks)]
    sizes = [h.size for h in per_rank[0]]
    for r in range(1, nranks):  # same shapes on every rank, own values
        per_rank[r] = [np.resize(h, n) for h, n in zip(per_rank[r], sizes)]

    def body(rank, comm):
        ex = A.GradientExchange(A.parse_spec(label), mode=mode, op=op, check="sync", comm=comm)
        ts = _to_device(np.random.default_rng(rank), per_rank[rank], cuda)
        ex(ts)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for t in ts]

    res = run_virtual_ranks(nranks, body)
    fn = O.exchange_allgather if mode == "allgather" else O.exchange_two_round
    want = fn(per_rank, kind, norm, dec, op)
    for r in range(nranks):
        for i, (a, b) in enumerate(zip(res[r], want)):
            assert a.tobytes() == b.tobytes(), (label, mode, op, nranks, r, i)


@pytest.mark.parametrize("case", range(9))
def test_blocked_matches_oracle(cuda, case):
    """Per-block max-abs (not a reference feature: encode_buffer applied to
    every block alone, oracle.encode_blocked): random sizes, block sizes,
    magnitudes per region (all-zero and subnormal blocks included)."""
    rng = np.random.default_rng(9600 + case)
    block = (1024, 2048, 4096)[case % 3]
    kind = ("dynamic-tree", "linear")[case % 2]
    n = int(np.exp(rng.uniform(np.log(1), np.log(3_000_000))))
    x = np.zeros(n, np.float32)
    pos = 0
    while pos < n:  # regions of random length and magnitude
        m = int(rng.integers(1, 3 * block))
        mag = float(rng.choice([0.0, 1e-42, 1e-3, 1.0, 1e20, 10.0 ** rng.uniform(-30, 30)]))
        x[pos:pos + m] = (rng.standard_normal(min(m, n - pos)) * mag).astype(np.float32)
        pos += m
    (xd,) = _to_device(rng, [x], cuda)
    cb = A.build_codebook(A.DataTypeSpec(kind, "absmax"))
    q = A.encode_buffer(xd, cb, block_size=block)
    codes = q.codes.view(-1).cpu().numpy()
    scales = q.block_scales.view(-1).cpu().numpy()
    y = A.decode_buffer(q, cb).view(-1).cpu().numpy()
    for b, b0 in enumerate(range(0, n, block)):
        c, s = O.c_encode(x[b0:b0 + block], kind, "absmax")
        assert codes[b0:b0 + block].tobytes() == c.tobytes(), (block, b)
        assert np.float32(scales[b]) == np.float32(s), (block, b)
        assert y[b0:b0 + block].tobytes() == O.c_decode(c, s, kind).tobytes(), (block, b)


@pytest.mark.parametrize("case", range(6))
def test_premax_exchange_matches_oracle(cuda, case):
    """Producer-fused maxima (scale_absmax_: y = fl(alpha x) and max|y|) and
    the one-pass encode: the same bits as the oracle's round trip of y."""
    rng = np.random.default_rng(9400 + case)
    label = ("dynamic-tree/absmax", "linear/absmax")[case % 2]
    kind, norm, dec = _oracle_args(label)
    host = _draw(rng, int(rng.integers(1, 20)), 12_000_000 if case < 2 else 2_000_000)
    alpha = float(np.float32(rng.choice([1.0, 0.5, 0.125, 1 / 3])))
    grads = _to_device(rng, host, cuda)
    outs = [torch.empty_like(g) for g in grads]
    ex = A.GradientExchange(A.parse_spec(label), check="sync")
    ex(grads, out=outs, amax=A.scale_absmax_(grads, alpha))
    for h, o in zip(host, outs):
        y = (h * np.float32(alpha)).astype(np.float32)
        c, s = O.c_encode(y, kind, norm, dec)
        assert o.cpu().numpy().tobytes() == O.c_decode(c, s, kind).tobytes(), (alpha, h.size)
