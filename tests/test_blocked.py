"""Per-block max-abs codec (north star "optional per-block max-abs"; not a
reference feature).  Parity target: the reference's encode_buffer applied to
each block alone (oracle.encode_blocked), bit for bit; decode is
table[c] * s_block (codecs.py:281)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1511_04561_b200 as A
from helpers import O


def test_oracle_blocked_is_per_block_reference_encode():
    x = O.sample_normal(10_000, 5)
    codes, scales = O.encode_blocked(x, "dynamic-tree", 4096)
    assert scales.shape == (3,)
    for b in range(3):
        c, s = O.encode(x[b * 4096:(b + 1) * 4096], "dynamic-tree", "absmax")
        assert np.array_equal(codes[b * 4096:(b + 1) * 4096], c) and scales[b] == np.float32(s)
    y = O.decode_blocked(codes, scales, "dynamic-tree", 4096)
    assert y.dtype == np.float32 and y.size == x.size


def test_blocked_symbols_exported():
    from paper_1511_04561_b200 import _native as N

    assert callable(N.lib.a8_encode_blocked) and callable(N.lib.a8_decode_blocked)


@pytest.mark.gpu
@pytest.mark.parametrize("block", [1024, 2048, 4096])
@pytest.mark.parametrize("n", [1, 17, 1024, 4095, 4096, 4097, 100_003, 1 << 20])
@pytest.mark.parametrize("kind", ["dynamic-tree", "linear"])
def test_blocked_codes_and_decode_match_oracle(cuda, block, n, kind):
    x = O.sample_normal(n, n + block, 0.0, 0.3)
    x[::7] *= 1e-3  # blocks with very different ranges
    x[5::11] = 0.0
    cb = A.build_codebook(A.DataTypeSpec(kind, "absmax"))
    q = A.encode_buffer(torch.from_numpy(x).to(cuda), cb, block_size=block)
    want_c, want_s = O.encode_blocked(x, kind, block)
    assert np.array_equal(q.codes.cpu().numpy(), want_c)
    assert np.array_equal(q.block_scales.cpu().numpy(), want_s)
    y = A.decode_buffer(q, cb).cpu().numpy().ravel()
    assert y.tobytes() == O.decode_blocked(want_c, want_s, kind, block).tobytes()


@pytest.mark.gpu
def test_blocked_edge_cases(cuda):
    cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
    z = torch.zeros(5000, device=cuda)
    q = A.encode_buffer(z, cb, block_size=4096)
    assert q.block_scales.cpu().tolist() == [1.0, 1.0]  # all-zero block -> scale 1 (codecs.py:240)
    assert int(q.codes.cpu().numpy().max()) == 0
    e = A.encode_buffer(torch.zeros(0, device=cuda), cb, block_size=1024)
    assert e.codes.numel() == 0 and e.block_scales.numel() == 0
    with pytest.raises(A.UsageError):
        _ = q.scale
    x = torch.randn(9000, device=cuda)
    x[8191] = float("inf")
    with pytest.raises(A.InputError):
        A.encode_buffer(x, cb, block_size=2048)
    with pytest.raises(A.ConfigError):
        A.encode_buffer(x, A.build_codebook(A.DataTypeSpec("mantissa", "decade", 1)), block_size=4096)
    with pytest.raises(A.ConfigError):
        A.encode_buffer(x, cb, block_size=3000)


@pytest.mark.gpu
def test_blocked_beyond_2_to_31_elements(cuda):
    """Per-block codec at 2^31 + 4099 elements: x repeats a seeded 2^20
    base (a whole number of blocks), so codes, block scales and decoded
    values repeat the base's, which are checked against the oracle."""
    P, reps, tail, block = 1 << 20, 2048, 4099, 4096
    base_np = O.sample_normal(P, 33, 0.0, 0.3)
    base_np[::7] *= 1e-3
    cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
    base = torch.from_numpy(base_np).to(cuda)
    qb = A.encode_buffer(base, cb, block_size=block)
    want_c, want_s = O.encode_blocked(base_np, "dynamic-tree", block)
    assert np.array_equal(qb.codes.cpu().numpy(), want_c)
    assert np.array_equal(qb.block_scales.cpu().numpy(), want_s)
    x = torch.empty(P * reps + tail, device=cuda)
    x[:P * reps].view(reps, P).copy_(base.expand(reps, P))
    x[P * reps:] = base[:tail]
    q = A.encode_buffer(x, cb, block_size=block)
    nb = P // block
    c, s = q.codes.view(-1), q.block_scales.view(-1)
    assert bool((c[:P * reps].view(reps, P) == qb.codes.view(1, P)).all())
    assert bool((s[:nb * reps].view(reps, nb) == qb.block_scales.view(1, nb)).all())
    tq = A.encode_buffer(base[:tail].clone(), cb, block_size=block)  # the ragged tail's blocks
    assert torch.equal(c[P * reps:], tq.codes.view(-1))
    assert torch.equal(s[nb * reps:], tq.block_scales.view(-1))
    del x
    y = A.decode_buffer(q, cb).view(-1)
    db = A.decode_buffer(qb, cb).view(-1)
    bad = y[:P * reps].view(reps, P) != db.view(1, P)
    if bool(bad.any()):  # report where (one intermittent failure seen in round 2, not reproduced)
        idx = bad.nonzero()[:8].tolist()
        flat = [r * P + c for r, c in idx]
        pytest.fail(f"{int(bad.sum())} decoded values differ; first at {flat} (chunks "
                    f"{sorted({f // 4096 for f in flat})}): got {[y[f].item() for f in flat[:3]]}, "
                    f"want {[db[f % P].item() for f in flat[:3]]}")
    del y, q, c, s
    torch.cuda.empty_cache()


# constants of a8_blocked.cu's streaming encode (guess-and-verify)
G_KEY0, G_LEN, G_MARGIN = 0x3400, 0x3F80 - 0x3400 + 1, 2.0 ** -18


def _guess_table(kind):
    v = O.book(kind).values
    mid = 0.5 * (v[:-1] + v[1:])
    yk = (((np.arange(G_LEN) + G_KEY0).astype(np.uint32)) << 16).view(np.float32).astype(np.float64)
    return np.searchsorted(mid * (1.0 + G_MARGIN), yk, side="left").astype(np.uint8), mid


@pytest.mark.parametrize("kind", ["dynamic-tree", "linear"])
def test_guess_buckets_hold_at_most_one_midpoint(kind):
    """The streaming per-block encode guesses c from the normalised value's
    bucket and verifies ONE threshold; that needs every bucket, widened by
    the normalisation's rounding (2^-22) and the margin, to hold at most one
    midpoint of the codebook."""
    G, mid = _guess_table(kind)
    lo = (((np.arange(G_LEN) + G_KEY0).astype(np.uint32)) << 16).view(np.float32).astype(np.float64)
    hi = (((np.arange(G_LEN) + G_KEY0 + 1).astype(np.uint32)) << 16).view(np.float32).astype(np.float64)
    w = 2.0 ** -22
    a = np.searchsorted(mid, lo * (1 - w) / (1 + G_MARGIN), side="left")
    b = np.searchsorted(mid, hi * (1 + w) * (1 + G_MARGIN), side="right")
    assert (b - a).max() <= 1
    assert mid[0] > 2.0 ** -23  # nothing below the table's first key


@pytest.mark.parametrize("kind", ["dynamic-tree", "linear"])
def test_guess_verify_restated_matches_reference(kind):
    """The kernel's per-element arithmetic restated in NumPy (float32
    normalisation, guess table, exact threshold verify) on blocks with
    random scales and elements at every threshold and its neighbours."""
    G, _ = _guess_table(kind)
    rng = np.random.default_rng(11)
    for trial in range(40):
        s = np.float32(np.exp(rng.uniform(np.log(2.0 ** -90), np.log(2.0 ** 90))))
        T = O.thresholds(kind, float(s))
        fin = T[T < 0x7F800000]
        near = np.concatenate([fin - 1, fin, fin + 1]).astype(np.uint32)
        mags = np.concatenate([near, rng.integers(0, int(np.float32(s).view(np.uint32)) + 1, 3000)]).astype(np.uint32)
        mags = mags[mags <= np.float32(s).view(np.uint32)]
        x = mags.view(np.float32).copy()
        x[::3] *= -1
        x = np.concatenate([x, [s]]).astype(np.float32)
        ref, rs = O.encode(x, kind, "absmax")
        assert np.float32(rs) == s
        r = np.float32(1.0) / s
        y = (np.abs(x) * r).astype(np.float32)
        key = (y.view(np.uint32) >> 16).astype(np.int64)
        c = G[np.maximum(key - G_KEY0, 0)].astype(np.int64)
        Tp = np.append(T, 0x7F800000)
        p = c + ((x.view(np.uint32) & 0x7FFFFFFF) >= Tp[c])
        code = (p | np.where((x < 0) & (p != 0), 0x80, 0)).astype(np.uint8)
        assert np.array_equal(code, ref), trial


@pytest.mark.gpu
@pytest.mark.parametrize("block", [2048, 4096])
def test_blocked_decode_staged_kernel_edges(cuda, block):
    """The staged per-block decode (full 4096-element chunks, aligned) plus
    the register kernel for the ragged tail and for unaligned outputs."""
    n = 4096 * 37 + 1234
    x = torch.randn(n, device=cuda) * 1e-2
    cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
    q = A.encode_buffer(x, cb, block_size=block)
    y = A.decode_buffer(q, cb)
    codes = q.codes_device.cpu().numpy()
    scales = q.block_scales.cpu().numpy()
    ref = np.empty(n, dtype=np.float32)
    tab = np.asarray(O.book("dynamic-tree").table, dtype=np.float32)
    for j in range(len(scales)):
        sl = slice(j * block, min(n, (j + 1) * block))
        ref[sl] = (tab[codes[sl]] * np.float32(scales[j])).astype(np.float32)
    assert y.cpu().numpy().tobytes() == ref.tobytes()
    buf = torch.empty(n + 1, device=cuda)  # an output 4 bytes off 16-byte alignment
    out = buf[1:]
    A.decode_buffer(q, cb, out=out)
    assert out.cpu().numpy().tobytes() == ref.tobytes()
