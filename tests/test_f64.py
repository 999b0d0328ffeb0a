"""float64 inputs: the reference computes them in float64 (codecs.py:254),
e.g. its DP/MP seams (mlp.py:330).  Goldens are reference codes for float64
data float32 cannot represent (incl. exact float64 midpoints)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O, golden, parse_tag

import paper_1511_04561_b200 as A


def f64_cases():
    g, meta = golden()
    for key in sorted(g.files):
        if key.startswith("f64/") and key.endswith("/x"):
            t = key[4:-2]
            yield t, parse_tag(t), g[key], g[f"f64/{t}/codes"], meta["f64"][t]["scale"]


@pytest.mark.parametrize("case", list(f64_cases()), ids=lambda c: c[0])
def test_oracle_float64_matches_reference(case):
    _, spec, x, ref, s = case
    codes, gs = O.encode(x, *spec)
    assert np.array_equal(codes, ref) and gs == s


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(f64_cases()), ids=lambda c: c[0])
def test_gpu_float64_matches_reference(case, cuda):
    _, spec, x, ref, s = case
    cb = A.build_codebook(A.DataTypeSpec(*spec))
    for inp in (x, torch.from_numpy(x).to(cuda)):
        q = A.encode_buffer(inp, cb)
        assert np.array_equal(q.codes_numpy(), ref)
        assert isinstance(q.codes, np.ndarray) == isinstance(inp, np.ndarray)  # NumPy in -> NumPy codes
        assert q.scale == s


@pytest.mark.gpu
def test_gpu_float64_edge_cases(cuda):
    cb = A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax"))
    with pytest.raises(A.InputError):
        A.encode_buffer(np.array([0.5, np.nan]), cb)
    q = A.encode_buffer(np.zeros(5), cb)
    assert q.scale == 1.0 and int(q.codes.max()) == 0
    assert A.encode_buffer(np.empty((0, 2)), cb).scale == 1.0
    # the reference seam: decode(encode(float64)) as float64 (mlp.py:170)
    rng = np.random.default_rng(2)
    x = rng.normal(size=(128, 1200)) * 1e-3
    y = A.roundtrip(x, cb.spec)
    assert y.dtype == np.float32
    assert y.tobytes() == O.roundtrip(x, "dynamic-tree", "absmax").astype(np.float32).tobytes()
    # multi-chunk absmax with the peak in the last chunk
    x = rng.normal(size=3 * 4096 + 11)
    x[-1] = 9.0
    assert np.array_equal(A.encode_buffer(x, cb).codes, O.encode(x, "dynamic-tree", "absmax")[0])
