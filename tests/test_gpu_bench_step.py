"""The bench's exact N = 1 step, parity-pinned at full config 3.

bench.py times ``GradientExchange(dynamic-tree/absmax, graph=True)`` over the
16 AlexNet-shaped gradients of ``bench.alexnet_grads(0)`` (61,100,840
elements) into ``out=`` tensors.  Here the same call (eager, graph-captured
and replayed) is checked element for element against the C oracle's round
trip of every tensor (oracle/approx8_oracle.c, the restatement of
codecs.py:244-288 pinned to the reference goldens): bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O

import paper_1511_04561_b200 as A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    import bench

    host = bench.alexnet_grads(0)
    want = []
    for g in host:
        c, s = O.c_encode(g.reshape(-1), "dynamic-tree", "absmax")
        want.append(O.c_decode(c, s, "dynamic-tree"))
    return host, want


@pytest.mark.parametrize("graph", [False, True])
def test_bench_step_matches_oracle(cuda, c3, graph):
    host, want = c3
    grads = [torch.from_numpy(g).to(cuda) for g in host]
    outs = [torch.empty_like(g) for g in grads]
    ex = A.GradientExchange(A.parse_spec("dynamic-tree/absmax"), mode="allgather", op="avg", check="deferred",
                            graph=graph)
    for _ in range(3):  # graph mode: eager first call, capture, then replays
        for o in outs:
            o.fill_(float("nan"))
        ex(grads, out=outs)
        ex.synchronize()
        for o, w in zip(outs, want):
            assert o.reshape(-1).cpu().numpy().tobytes() == w.tobytes()
    # the inputs are untouched (out= given)
    for g, h in zip(grads, host):
        assert g.cpu().numpy().tobytes() == h.tobytes()


def test_bench_step_premax_matches_oracle(cuda, c3):
    """The one-pass path of bench.py's codec_sweep.premax on the same data."""
    host, want = c3
    grads = [torch.from_numpy(g).to(cuda).reshape(-1) for g in host]
    outs = [torch.empty_like(g) for g in grads]
    ex = A.GradientExchange(A.parse_spec("dynamic-tree/absmax"), check="sync")
    m = A.scale_absmax_(grads, 1.0)
    assert np.array_equal(m.cpu().numpy(), np.array([np.abs(g).max() for g in host], dtype=np.float32))
    ex(grads, out=outs, amax=m)
    for o, w in zip(outs, want):
        assert o.cpu().numpy().tobytes() == w.tobytes()
