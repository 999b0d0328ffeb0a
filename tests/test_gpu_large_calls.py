"""Large absmax calls (beyond the resident kernel's shared-memory capacity)
through the ticket encode kernel: segments of one chunk or a ragged last
chunk, empty segments, many small segments between large ones, a segment
whose bucket table is invalid (threshold search), all-zero and subnormal
segments, non-finite input and recovery.  Every case is checked element for
element against the C oracle's round trip (oracle/approx8_oracle.c, the
restatement of codecs.py:244-288).

(Written for the grid-barrier encode experiment, whose kernel
was not kept; the cases stay as coverage of the product kernel.)
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu


def _check(cuda, sizes, kind="dynamic-tree", seed=0, scales=None):
    rng = np.random.default_rng(seed)
    host = []
    for i, n in enumerate(sizes):
        s = 1e-3 if scales is None else scales[i % len(scales)]
        host.append((rng.standard_normal(n) * s).astype(np.float32))
    grads = [torch.from_numpy(h).to(cuda) for h in host]
    outs = [torch.empty_like(g).fill_(float("nan")) for g in grads]
    ex = A.GradientExchange(A.DataTypeSpec(kind, "absmax"), check="sync")
    ex(grads, out=outs)
    for h, o in zip(host, outs):
        c, s = O.c_encode(h, kind, "absmax")
        want = O.c_decode(c, s, kind)
        assert o.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("kind", ["dynamic-tree", "linear"])
def test_mixed_segments(cuda, kind):
    # 8.3M elements: beyond the resident kernel; ragged last chunks, single
    # chunks, an empty segment, and runs that straddle CTA ranges
    sizes = [5_000_004, 8, 0, 12_288, 4_100, 1_228_796, 2_000_000, 36, 4_096]
    _check(cuda, sizes, kind)


def test_many_small_between_large(cuda):
    sizes = []
    for i in range(14):
        sizes += [700_000 + 4 * i, 4 * (i + 1), 4_096 * (i % 3) + 12]
    _check(cuda, sizes[:32], seed=3, scales=[1e-3, 10.0, 1e-20])


def test_wide_dynamic_range(cuda):
    # a segment whose table is invalid (too many buckets): threshold search
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(9_000_000) * np.exp(rng.uniform(-40, 40, 9_000_000))).astype(np.float32)
    g = torch.from_numpy(x).to(cuda)
    out = torch.empty_like(g)
    A.GradientExchange(A.DataTypeSpec("dynamic-tree", "absmax"), check="sync")([g], out=[out])
    c, s = O.c_encode(x, "dynamic-tree", "absmax")
    assert out.cpu().numpy().tobytes() == O.c_decode(c, s, "dynamic-tree").tobytes()


def test_all_zero_and_tiny_values(cuda):
    sizes = [3_000_000, 3_000_000, 3_000_000]
    host = [np.zeros(sizes[0], np.float32), np.full(sizes[1], 1e-42, np.float32),
            np.random.default_rng(1).standard_normal(sizes[2]).astype(np.float32)]
    grads = [torch.from_numpy(h).to(cuda) for h in host]
    outs = [torch.empty_like(g) for g in grads]
    A.GradientExchange(A.DataTypeSpec("dynamic-tree", "absmax"), check="sync")(grads, out=outs)
    for h, o in zip(host, outs):
        c, s = O.c_encode(h, "dynamic-tree", "absmax")
        assert o.cpu().numpy().tobytes() == O.c_decode(c, s, "dynamic-tree").tobytes()


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_non_finite_raises_and_recovers(cuda, bad):
    ex = A.GradientExchange(A.DataTypeSpec("dynamic-tree", "absmax"), check="sync")
    grads = [torch.randn(6_000_000, device=cuda), torch.randn(4_000_000, device=cuda)]
    outs = [torch.empty_like(g) for g in grads]
    grads[1][3_999_999] = bad
    with pytest.raises(A.InputError):
        ex(grads, out=outs)
    grads[1][3_999_999] = 0.5
    ex(grads, out=outs)  # the workspace was left clean
    for g, o in zip(grads, outs):
        h = g.cpu().numpy()
        c, s = O.c_encode(h, "dynamic-tree", "absmax")
        assert o.cpu().numpy().tobytes() == O.c_decode(c, s, "dynamic-tree").tobytes()


def test_encode_buffer_codes(cuda):
    """encode_buffer (one tensor, codes + scale) through the same kernel."""
    x = (np.random.default_rng(11).standard_normal(16_000_004) * 3e-2).astype(np.float32)
    q = A.encode_buffer(torch.from_numpy(x).to(cuda), A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax")))
    c, s = O.c_encode(x, "dynamic-tree", "absmax")
    codes = q.codes.cpu().numpy() if hasattr(q.codes, "cpu") else np.asarray(q.codes)
    assert codes.tobytes() == c.tobytes()
    assert np.float32(q.scale) == np.float32(s)
