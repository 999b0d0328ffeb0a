"""GPU parity of the sm_100a codec against the reference goldens and the oracle.

Bar: codes bit-exact; scales bit-exact; decoded values bit-exact (a single
float32 round-to-nearest multiply, codecs.py:281).  Sizes run from the
reference's own cases up to BASELINE config sizes, where size-independent
properties (sign symmetry, idempotence, order, power-of-two invariance,
oracle agreement on large seeded inputs) are checked.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O, acceptance_inputs, fullrange_cases, golden, golden_cases, sha, tag

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu

ALL_SPECS = [("dynamic-tree", "none", 0), ("dynamic-tree", "absmax", 0), ("linear", "none", 0),
             ("linear", "absmax", 0), ("static-tree", "none", 0), ("static-tree", "decade", 1),
             ("mantissa", "none", 0), ("mantissa", "decade", 2), ("mantissa", "decade", -1)]


def S(spec):
    return A.DataTypeSpec(*spec)


def enc(x, spec, dev):
    cb = A.build_codebook(S(spec))
    q = A.encode_buffer(torch.from_numpy(np.ascontiguousarray(x)).to(dev), cb)
    return q.codes.cpu().numpy(), q.scale, q, cb


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0])
def test_codes_match_reference_vectors(case, cuda):
    name, spec, x, ref = case
    codes, s, q, cb = enc(x, spec, cuda)
    assert np.array_equal(codes, ref), f"{name}: {(codes != ref).sum()} mismatches"
    assert s == O.encode(x, *spec)[1]
    dec = A.decode_buffer(q, cb).cpu().numpy()
    assert dec.tobytes() == O.decode(ref, s, spec[0]).tobytes(), name


def test_fullrange_buffers(cuda):
    for base, spec, xs, cs, scales in fullrange_cases():
        for x, c, s in zip(xs, cs, scales):
            codes, gs, _, _ = enc(x, spec, cuda)
            assert np.array_equal(codes, c), base
            assert gs == s, base


def test_acceptance_100k_digests(cuda):
    """test_acceptance.py:116-129 inputs, compared by digest with the reference."""
    _, meta = golden()
    for spec, x in acceptance_inputs():
        m = meta["acceptance"][tag(spec)]
        codes, s, q, cb = enc(x, spec, cuda)
        assert sha(codes) == m["sha_codes"], tag(spec)
        assert s == m["scale"]
        assert sha(A.decode_buffer(q, cb).cpu().numpy()) == m["sha_decoded"], tag(spec)


def test_config1_digests(cuda):
    """BASELINE config 1: errorbench.sample(normal, 2**20, seed 0)."""
    _, meta = golden()
    x = O.sample_normal(2**20, 0)
    for t, m in meta["c1"].items():
        if t == "sha_x":
            continue
        kind, norm = t.split("/")
        spec = (kind, "decade", int(norm[6:])) if norm.startswith("decade") else (kind, norm, 0)
        codes, s, q, cb = enc(x, spec, cuda)
        assert sha(codes) == m["sha_codes"], t
        assert s == m["scale"], t
        assert sha(A.decode_buffer(q, cb).cpu().numpy()) == m["sha_decoded"], t


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 15, 16, 17, 63, 1000, 4095, 4096, 4097, 8191, 12289,
                               65536 + 7, 2**20 + 3])
@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[3], ALL_SPECS[5], ALL_SPECS[7]], ids=tag)
def test_sizes_and_tails(n, spec, cuda):
    rng = np.random.default_rng(n)
    x = (rng.normal(size=n) * 10.0 ** rng.integers(-6, 2, size=n)).astype(np.float32)
    codes, s, q, cb = enc(x, spec, cuda)
    ref, rs = O.encode(x, *spec)
    assert s == rs
    assert np.array_equal(codes, ref)
    assert A.decode_buffer(q, cb).cpu().numpy().tobytes() == O.decode(ref, s, spec[0]).tobytes()


@pytest.mark.parametrize("spec", ALL_SPECS, ids=tag)
def test_peak_position_and_misaligned_views(spec, cuda):
    rng = np.random.default_rng(11)
    base = rng.normal(size=3 * 4096 + 50).astype(np.float32)
    for pos in (0, 4095, 4096, 12287, base.size - 1):
        x = base.copy()
        x[pos] = -7.5  # the peak in different chunks, including the tail
        codes, s, _, _ = enc(x, spec, cuda)
        assert np.array_equal(codes, O.encode(x, *spec)[0]), pos
    t = torch.from_numpy(base).to(cuda)
    for off in (1, 2, 3, 5):  # not 16-byte aligned: scalar path
        v = t[off:]
        cb = A.build_codebook(S(spec))
        q = A.encode_buffer(v, cb)
        assert np.array_equal(q.codes.cpu().numpy(), O.encode(base[off:], *spec)[0]), off


def test_empty_zero_and_shape(cuda):
    cb = A.build_codebook(A.DataTypeSpec("linear", "absmax"))
    q = A.encode_buffer(torch.empty((0, 3), device=cuda), cb)
    assert q.codes.numel() == 0 and q.scale == 1.0
    assert tuple(A.decode_buffer(q, cb).shape) == (0, 3)
    cbd = A.build_codebook(A.DataTypeSpec("mantissa", "decade", 2))
    assert A.encode_buffer(torch.empty(0, device=cuda), cbd).scale == np.float32(100.0)
    for spec in ALL_SPECS:
        cb = A.build_codebook(S(spec))
        q = A.encode_buffer(torch.zeros(4097, device=cuda), cb)
        assert int(q.codes.max()) == 0
        if spec[1] == "absmax":
            assert q.scale == 1.0
        assert float(A.decode_buffer(q, cb).abs().max()) == 0.0
    cb = A.build_codebook(A.DataTypeSpec("mantissa"))
    x = torch.randn(3, 4, 5, device=cuda)
    q = A.encode_buffer(x, cb)
    assert q.shape == (3, 4, 5) and tuple(A.decode_buffer(q, cb).shape) == (3, 4, 5)


@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[2], ALL_SPECS[5]], ids=tag)
@pytest.mark.parametrize("pos", [0, 3, 4096 + 17, 3 * 4096 + 2])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), float("-inf")])
def test_non_finite_raises_input_error(spec, pos, bad, cuda):
    x = torch.randn(3 * 4096 + 5, device=cuda)
    x[pos] = bad
    cb = A.build_codebook(S(spec))
    with pytest.raises(A.InputError):
        A.encode_buffer(x, cb)
    # the next call on the same workspace is clean again
    q = A.encode_buffer(torch.ones(8, device=cuda), cb)
    assert q.scale > 0


def test_spec_mismatch_raises_usage_error(cuda):
    cb_lin = A.build_codebook(A.DataTypeSpec("linear"))
    cb_dyn = A.build_codebook(A.DataTypeSpec("dynamic-tree"))
    q = A.encode_buffer(torch.tensor([0.5], device=cuda), cb_lin)
    with pytest.raises(A.UsageError):
        A.decode_buffer(q, cb_dyn)


def test_tie_breaks_toward_smaller_and_table_identity(cuda):
    cb = A.build_codebook(A.DataTypeSpec("linear"))
    mid = float(cb.sorted_values[1]) / 2.0
    q = A.encode_buffer(torch.tensor([mid, -mid], device=cuda), cb)
    assert q.codes.tolist() == [0, 0]
    for kind in ("dynamic-tree", "static-tree", "linear", "mantissa"):
        spec = A.DataTypeSpec(kind)
        v = torch.from_numpy(A.build_codebook(spec).decode_table.copy()).to(cuda)
        assert torch.equal(A.roundtrip(v, spec), v), kind


@pytest.mark.parametrize("spec", ALL_SPECS, ids=tag)
def test_properties_on_random_buffers(spec, cuda):
    """test_properties.py:50-102 invariants on many random buffers."""
    rng = np.random.default_rng(hash(tag(spec)) % 2**32)
    cb = A.build_codebook(S(spec))
    for n in (1, 7, 24, 333, 5000):
        x = (rng.normal(size=n) * 10.0 ** rng.integers(-8, 3, size=n)).astype(np.float32)
        t = torch.from_numpy(x).to(cuda)
        pos = A.encode_buffer(t, cb).codes
        neg = A.encode_buffer(-t, cb).codes
        zero = pos == 0
        assert torch.equal(neg[zero], pos[zero]) and torch.equal(neg[~zero], pos[~zero] ^ 0x80)
        assert torch.equal(A.encode_buffer(t.clone(), cb).codes, pos)  # purity
        srt = torch.sort(t).values
        d = A.roundtrip(srt, cb.spec)
        assert bool((d[1:] >= d[:-1]).all())  # order preservation
        if spec[1] != "absmax":
            once = A.roundtrip(t, cb.spec)
            assert torch.equal(A.roundtrip(once, cb.spec), once)  # idempotence
        else:
            for f in (0.25, 2.0, 1024.0):
                assert torch.equal(A.encode_buffer(t * f, cb).codes, pos)


@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[3], ALL_SPECS[5], ALL_SPECS[7]], ids=tag)
def test_large_seeded_buffer_matches_oracle(spec, cuda):
    """2^24 + 5 elements (multi-wave persistent grid) vs the oracle."""
    x = O.sample_normal(2**24 + 5, 7, 0.0, 0.01)
    codes, s, q, cb = enc(x, spec, cuda)
    ref, rs = O.encode(x, *spec)
    assert s == rs
    assert np.array_equal(codes, ref)


def test_roundtrip_numpy_in_numpy_out(cuda):
    x = O.sample_normal(10000, 1)
    y = A.roundtrip(x, A.DataTypeSpec("dynamic-tree", "absmax"))
    assert isinstance(y, np.ndarray) and y.dtype == np.float32
    assert y.tobytes() == O.roundtrip(x, "dynamic-tree", "absmax").tobytes()


def test_error_suite_cells_on_gpu(cuda):
    """Error bench cells (errorbench.py:79-99) from GPU round trips equal the
    reference's published-protocol numbers exactly."""
    _, meta = golden()
    cells = {(c["seed"]): c for c in meta["suite"]}
    for seed, kind, spec in [(0, "dynamic-tree", ("dynamic-tree", "absmax", 0)),
                             (1, "linear", ("linear", "absmax", 0)),
                             (6, "mantissa", ("mantissa", "decade", 1)),
                             (11, "static-tree", ("static-tree", "decade", 2))]:
        c = cells[seed]
        assert c["spec"] == tag(spec)
        d_idx = seed // 4
        sigma = [None, 1.0, 10.0, 0.2][d_idx]
        x = O.sample_uniform01(1_000_000, seed) if d_idx == 0 else O.sample_normal(1_000_000, seed, 0.0, sigma)
        y = A.roundtrip(x, S(spec)).astype(np.float64)
        x64 = x.astype(np.float64)
        err = np.abs(x64 - y)
        nz = x64 != 0
        assert float(err.mean()) == c["mean_abs_error"]
        assert float(np.mean(err[nz] / np.abs(x64[nz])) * 100.0) == c["mean_rel_error_pct"]


@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[5]], ids=tag)
@pytest.mark.parametrize("bad", [float("nan"), float("-inf")])
def test_non_finite_in_large_call_ticket_kernel(spec, bad, cuda):
    """Beyond the resident kernel's capacity the ticket kernel runs: a
    non-finite value inside a full, aligned chunk (fast path) must still
    raise, and the workspace must be clean for the next call."""
    x = torch.randn(8_000_000, device=cuda)
    x[5_000_003] = bad
    cb = A.build_codebook(S(spec))
    with pytest.raises(A.InputError):
        A.encode_buffer(x, cb)
    x[5_000_003] = 0.0
    q = A.encode_buffer(x, cb)
    assert q.scale > 0


@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[3], ALL_SPECS[5], ALL_SPECS[6]], ids=tag)
@pytest.mark.parametrize("n", [1, 5, 4096, 100_003, 2_000_000, 8_000_000])
def test_roundtrip_fused_and_fallback_match_oracle(spec, n, cuda):
    """roundtrip(): one fused kernel (a8_roundtrip) up to the resident
    capacity, encode + decode beyond it (8M) -- both equal the reference
    round trip bit for bit; NumPy in -> NumPy out, torch in -> torch out."""
    rng = np.random.default_rng(n)
    x = (rng.normal(0, 0.05, size=n)).astype(np.float32)
    x[::9] = 0.0
    want = O.roundtrip(x, *spec)
    got = A.roundtrip(x, S(spec), device=cuda)
    assert isinstance(got, np.ndarray) and got.tobytes() == want.tobytes()
    gt = A.roundtrip(torch.from_numpy(x).to(cuda), S(spec))
    assert isinstance(gt, torch.Tensor) and gt.cpu().numpy().tobytes() == want.tobytes()


def test_roundtrip_fused_non_finite_and_shapes(cuda):
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    x = torch.randn(3, 5, 7, device=cuda)
    y = A.roundtrip(x, spec)
    assert y.shape == x.shape
    assert y.cpu().numpy().tobytes() == O.roundtrip(x.cpu().numpy(), "dynamic-tree", "absmax").tobytes()
    x[1, 2, 3] = float("nan")
    with pytest.raises(A.InputError):
        A.roundtrip(x, spec)
    y2 = A.roundtrip(torch.randn(100, device=cuda), spec)  # clean afterwards
    assert torch.isfinite(y2).all()


@pytest.mark.parametrize("spec", [ALL_SPECS[1], ALL_SPECS[7]], ids=tag)
def test_beyond_2_to_31_elements(spec, cuda):
    """Maximum sizes: a buffer of 2^31 + 4099 elements (8.6 GB, 64-bit
    indexing everywhere).  x repeats a seeded 2^20-element base (whose codes
    are checked against the oracle) 2048 times plus a ragged tail, so the
    scale is the base's and every period's codes and decoded values must
    equal the base's."""
    P, reps, tail = 1 << 20, 2048, 4099
    base_np = O.sample_normal(P, 31, 0.0, 0.01)
    ref, rs = O.encode(base_np, *spec)
    cb = A.build_codebook(S(spec))
    base = torch.from_numpy(base_np).to(cuda)
    qb = A.encode_buffer(base, cb)
    assert np.array_equal(qb.codes.cpu().numpy(), ref) and qb.scale == rs
    db = A.decode_buffer(qb, cb)
    x = torch.empty(P * reps + tail, device=cuda)
    x[:P * reps].view(reps, P).copy_(base.expand(reps, P))
    x[P * reps:] = base[:tail]
    q = A.encode_buffer(x, cb)
    assert q.scale == rs
    c = q.codes.view(-1)
    assert bool((c[:P * reps].view(reps, P) == qb.codes.view(1, P)).all())
    assert torch.equal(c[P * reps:], qb.codes[:tail])
    del x
    y = A.decode_buffer(q, cb).view(-1)
    assert bool((y[:P * reps].view(reps, P) == db.view(1, P)).all())
    assert torch.equal(y[P * reps:], db[:tail])
    del y, q, c
    torch.cuda.empty_cache()


def test_numpy_in_numpy_out(cuda):
    """Drop-in types (codecs.py:207-282): NumPy input gives NumPy uint8 codes
    and a NumPy float32 decode of the input's shape; the reference's callers
    (mlp.py:171 .astype, tensorfile.py:74 codes.astype) work on them."""
    x = O.sample_normal(3 * 4099, 4).reshape(3, 4099)
    for spec in (("dynamic-tree", "absmax"), ("mantissa", "decade", 1)):
        cb = A.build_codebook(A.DataTypeSpec(*spec))
        q = A.encode_buffer(x, cb)
        ref, s = O.encode(x.ravel(), *spec)
        assert isinstance(q.codes, np.ndarray) and q.codes.dtype == np.uint8
        assert np.array_equal(q.codes, ref) and q.scale == s
        assert q.codes.astype(np.uint8).tobytes() == ref.tobytes()
        y = A.decode_buffer(q, cb)
        assert isinstance(y, np.ndarray) and y.dtype == np.float32 and y.shape == x.shape
        assert y.tobytes() == O.decode(ref, s, spec[0]).reshape(x.shape).tobytes()
        assert y.astype(np.float64).dtype == np.float64
        # a QuantizedTensor built by a caller from NumPy parts (tensorfile.read_tensor)
        q2 = A.QuantizedTensor(codes=ref.copy(), shape=x.shape, spec=cb.spec, scale=s)
        assert A.decode_buffer(q2, cb).tobytes() == y.tobytes()
        # edits to the exposed codes are what decodes read
        q.codes[0] = cb.zero_code
        assert A.decode_buffer(q, cb).ravel()[0] == 0.0
    empty = A.encode_buffer(np.zeros((0, 4), np.float32), A.build_codebook(A.DataTypeSpec("linear", "absmax")))
    assert isinstance(empty.codes, np.ndarray) and empty.codes.size == 0 and empty.scale == 1.0
