"""1-bit error-feedback quantizer on the GPU vs the reference
(codecs.py:291-348; test_codecs.py:354-416, test_properties.py:105-120).

Goldens: 12 chained onebit_quantize steps of the real reference (bits, the
two float32 levels, the float64 residual after each step, the decoded
output).  The kernels reproduce them bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import golden

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu


def test_chained_steps_match_reference(cuda):
    g, _ = golden()
    st = A.OneBitState.zeros((3000,), device=cuda)
    for k in range(12):
        x = g[f"onebit/{k}/g"]
        q = A.onebit_quantize(torch.from_numpy(x).to(cuda), st)
        assert np.array_equal(q.codes.cpu().numpy(), g[f"onebit/{k}/bits"]), k
        assert (q.pos_level, q.neg_level) == tuple(g[f"onebit/{k}/levels"]), k
        assert st.residual.cpu().numpy().tobytes() == g[f"onebit/{k}/residual"].tobytes(), k
        assert A.onebit_decode(q).cpu().numpy().tobytes() == g[f"onebit/{k}/decoded"].tobytes(), k


def test_two_sided_means_and_packing(cuda):
    gg = torch.tensor([1.0, -1.0, 3.0, -5.0], dtype=torch.float64, device=cuda)
    st = A.OneBitState.zeros(gg.shape, device=cuda)
    q = A.onebit_quantize(gg, st)
    assert q.pos_level == pytest.approx(2.0) and q.neg_level == pytest.approx(-3.0)
    out = A.onebit_decode(q)
    assert torch.allclose(out.double(), torch.tensor([2.0, -3.0, 2.0, -3.0], device=cuda, dtype=torch.float64))
    assert torch.equal(st.residual, gg - out.double())
    q17 = A.onebit_quantize(torch.ones(17, device=cuda), A.OneBitState.zeros((17,), device=cuda))
    assert q17.nbits == 1 and q17.codes.numel() == 3 and tuple(A.onebit_decode(q17).shape) == (17,)
    c = torch.full((3, 3), 0.75, dtype=torch.float64, device=cuda)
    st3 = A.OneBitState.zeros((3, 3), device=cuda)
    assert torch.allclose(A.onebit_decode(A.onebit_quantize(c, st3)).double(), c)
    assert float(st3.residual.abs().max()) == 0.0


def test_errors(cuda):
    with pytest.raises(A.UsageError):
        A.onebit_quantize(torch.ones(5, device=cuda), A.OneBitState.zeros((4,), device=cuda))
    with pytest.raises(A.InputError):
        A.onebit_quantize(torch.tensor([1.0, float("nan")], device=cuda), A.OneBitState.zeros((2,), device=cuda))
    with pytest.raises(A.UsageError):
        A.onebit_decode(A.QuantizedTensor(np.zeros(1, np.uint8), (1,), A.DataTypeSpec("linear"), 1.0))


def test_residual_identity_and_telescoping(cuda):
    rng = np.random.default_rng(7)
    st = A.OneBitState.zeros((64,), device=cuda)
    tot_g = torch.zeros(64, dtype=torch.float64, device=cuda)
    tot_o = torch.zeros(64, dtype=torch.float64, device=cuda)
    for _ in range(100):
        x = torch.from_numpy(rng.normal(size=64)).to(cuda)
        prev = st.residual.clone()
        out = A.onebit_decode(A.onebit_quantize(x, st)).double()
        assert torch.equal(st.residual, (x + prev) - out)  # bit-exact residual identity
        tot_g += x
        tot_o += out
    assert torch.allclose(tot_g - tot_o, st.residual, atol=1e-9)


def test_large_tensor_bits_and_levels(cuda):
    """2^22 elements, multi-CTA partial sums: bits exact, levels within the
    float64-summation-order caveat (equal in practice)."""
    rng = np.random.default_rng(11)
    x = rng.normal(0, 1e-2, size=1 << 22).astype(np.float32)
    res = rng.normal(0, 1e-3, size=1 << 22)
    st = A.OneBitState(torch.from_numpy(res.copy()).to(cuda))
    q = A.onebit_quantize(torch.from_numpy(x).to(cuda), st)
    corrected = x.astype(np.float64) + res
    pos = corrected >= 0
    assert np.array_equal(q.codes.cpu().numpy(), np.packbits(pos))
    pl, nl = float(np.float32(corrected[pos].mean())), float(np.float32(corrected[~pos].mean()))
    assert q.pos_level == pl and q.neg_level == nl
    recon = np.where(pos, pl, nl)
    assert st.residual.cpu().numpy().tobytes() == (corrected - recon).tobytes()


def test_non_finite_leaves_state_untouched(cuda):
    """codecs.py:317-318 raises before touching the state."""
    rng = np.random.default_rng(5)
    st = A.OneBitState.zeros((5000,), device=cuda)
    A.onebit_quantize(torch.from_numpy(rng.normal(size=5000)).to(cuda), st)
    before = st.residual.clone()
    bad = torch.from_numpy(rng.normal(size=5000)).to(cuda)
    bad[4321] = float("inf")
    with pytest.raises(A.InputError):
        A.onebit_quantize(bad, st)
    assert torch.equal(st.residual, before)
    q = A.onebit_quantize(bad, st, sync=False)  # asynchronous: checked later
    with pytest.raises(A.InputError):
        q._finish()
    assert torch.equal(st.residual, before)


def test_host_state_numpy_in_numpy_out(cuda):
    """Reference types for host callers (mlp.py:313-321): NumPy residual,
    NumPy packbits codes, float levels, NumPy decode; chained goldens."""
    g, _ = golden()
    st = A.OneBitState.zeros((3000,))
    assert isinstance(st.residual, np.ndarray)
    for k in range(12):
        q = A.onebit_quantize(g[f"onebit/{k}/g"], st)
        assert isinstance(q.codes, np.ndarray) and np.array_equal(q.codes, g[f"onebit/{k}/bits"]), k
        assert (q.pos_level, q.neg_level) == tuple(g[f"onebit/{k}/levels"]), k
        assert isinstance(st.residual, np.ndarray)
        assert st.residual.tobytes() == g[f"onebit/{k}/residual"].tobytes(), k
        out = A.onebit_decode(q)
        assert isinstance(out, np.ndarray) and out.tobytes() == g[f"onebit/{k}/decoded"].tobytes(), k
    prev = st.residual.copy()
    with pytest.raises(A.InputError):
        A.onebit_quantize(np.full(3000, np.nan), st)
    assert np.array_equal(st.residual, prev)


def test_quantize_multi_bit_identical_to_per_tensor(cuda):
    """a8_onebit_quantize_multi (the 1-bit exchange's two launches for all
    tensors) gives each tensor exactly what a8_onebit_quantize gives it
    alone: bits, levels, status and the updated residual, over 3 chained
    steps, float32 and float64 inputs, empty and ragged tensors."""
    from paper_1511_04561_b200.exchange import CudaSegmentCodec, OneBitExchange

    sizes = [0, 1, 7, 8, 1000, 4097, 70001, 1 << 20, 3_000_001]
    rng = np.random.default_rng(3)
    codec = CudaSegmentCodec()
    offs, lev, st, P = OneBitExchange.layout(sizes)
    for dt in (torch.float32, torch.float64):
        ra = [torch.zeros(n, dtype=torch.float64, device=cuda) for n in sizes]
        rb = [torch.zeros(n, dtype=torch.float64, device=cuda) for n in sizes]
        for step in range(3):
            xs = [torch.from_numpy(rng.normal(size=n)).to(device=cuda, dtype=dt) for n in sizes]
            ba = torch.zeros(P, dtype=torch.uint8, device=cuda)
            bb = torch.zeros(P, dtype=torch.uint8, device=cuda)
            for i, x in enumerate(xs):
                codec.onebit_quantize(x, ra[i], ba, offs[i], lev + 8 * i, st + 4 * i)
            codec.onebit_quantize_many(xs, rb, bb, offs, [lev + 8 * i for i in range(len(sizes))],
                                       [st + 4 * i for i in range(len(sizes))])
            assert torch.equal(ba, bb), (dt, step)
            for a, b in zip(ra, rb):
                assert torch.equal(a, b), (dt, step)
