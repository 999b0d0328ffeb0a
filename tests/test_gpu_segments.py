"""Multi-segment encode/decode (one launch over many tensors) vs the oracle.

Exercises the persistent encode's ticket schedule (groups, held-back E tails,
per-CTA A-run flushes) and the multi-block code layout used by two_round.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O

import paper_1511_04561_b200 as A
from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan

pytestmark = pytest.mark.gpu


def encode_segments(xs, spec, dev, nblocks=1):
    """Encode `xs` in one a8_encode call into a flat (or N-block) slab; return
    per-segment codes and scales read back through the layout arithmetic."""
    plan = make_plan([x.size for x in xs], nblocks)
    L = plan.shard if nblocks > 1 else plan.flat
    B = L + plan.gap
    buf = torch.zeros(nblocks * B, dtype=torch.uint8, device=dev)
    ts = [torch.from_numpy(x).to(dev) for x in xs]
    cb = A.build_codebook(spec)
    CudaSegmentCodec().encode(ts, plan.offs, list(range(len(xs))), cb, buf, 0, L, L, B, B // 4, nblocks,
                              L + 4 * plan.status_slot)
    torch.cuda.synchronize()
    mem = buf.cpu().numpy()
    codes, scales = [], []
    for t, x in enumerate(xs):
        e = np.arange(x.size, dtype=np.int64) + plan.offs[t]
        codes.append(mem[(e // L) * B + e % L])
        scales.append(float(np.frombuffer(mem[L + 4 * t:L + 4 * t + 4].tobytes(), np.float32)[0]))
    status = int(np.frombuffer(mem[L + 4 * plan.status_slot:L + 4 * plan.status_slot + 4].tobytes(), np.uint32)[0])
    return codes, scales, status


def check(xs, spec, dev, nblocks=1):
    codes, scales, status = encode_segments(xs, spec, dev, nblocks)
    assert status == 0
    bad = []
    for t, (x, c, s) in enumerate(zip(xs, codes, scales)):
        ref, rs = O.encode(x, spec.kind.value, spec.normalization.value, spec.decades)
        if rs != s or not np.array_equal(c, ref):
            bad.append((t, x.size, s, rs, int((c != ref).sum())))
    assert not bad, bad


SPECS = [A.DataTypeSpec("dynamic-tree", "absmax"), A.DataTypeSpec("linear", "absmax"),
         A.DataTypeSpec("mantissa", "decade", 1)]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.label())
def test_many_small_segments(spec, cuda):
    rng = np.random.default_rng(1)
    xs = [(rng.normal(size=int(n)) * 10.0 ** rng.integers(-4, 2)).astype(np.float32)
          for n in rng.integers(0, 9000, size=40)]
    check(xs, spec, cuda)


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.label())
def test_group_boundaries_and_tails(spec, cuda):
    rng = np.random.default_rng(2)
    sizes = [5, 70000, 3 << 20, 1000, (2 << 20) + 17, 4096 * 3, 9 << 20]
    xs = [(rng.normal(size=n) * (1 + i)).astype(np.float32) for i, n in enumerate(sizes)]
    check(xs, spec, cuda)


@pytest.mark.parametrize("nblocks", [2, 3, 4, 8])
def test_multi_block_layout(nblocks, cuda):
    rng = np.random.default_rng(3)
    xs = [rng.normal(size=n).astype(np.float32) for n in (1200, 1, 17, 0, 300, 64, 5000, 70000, 123457)]
    for spec in SPECS:
        check(xs, spec, cuda, nblocks)


def test_decoded_values_reencode(cuda):
    """Re-encoding decoded averages (two_round round 2): inputs sit exactly on
    scaled table values and midpoints."""
    rng = np.random.default_rng(4)
    for spec in SPECS:
        g = [rng.normal(size=n).astype(np.float32) for n in (4096, 70000, 1000)]
        d = [O.roundtrip(x, spec.kind.value, spec.normalization.value, spec.decades) for x in g]
        avg = [((a + a[::-1]) / np.float32(2)).astype(np.float32) for a in d]
        check(d + avg, spec, cuda)


@pytest.mark.parametrize("with_status_in", [False, True])
def test_adjacent_slices_of_one_buffer(with_status_in, cuda):
    """two_round round-2 shape: pieces are adjacent 16-aligned slices of one
    shard buffer, encoded into a multi-block slab with a chained status."""
    rng = np.random.default_rng(5)
    sizes = [1200, 1, 17, 300, 64, 5000, 12544]
    offs = [0, 1200, 1216, 1248, 1552, 1616, 6624]
    L = 19168
    base = torch.from_numpy(rng.normal(size=L).astype(np.float32) * 1e-2).to(cuda)
    xs = [base[o:o + n] for o, n in zip(offs, sizes)]
    B = L + 64
    buf = torch.zeros(4 * B, dtype=torch.uint8, device=cuda)
    st_in = torch.zeros(1, dtype=torch.int32, device=cuda)
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    cb = A.build_codebook(spec)
    CudaSegmentCodec().encode(xs, offs, list(range(7)), cb, buf, 0, L, L, B, 0, 1, L + 4 * 16,
                              status_in=st_in if with_status_in else None)
    torch.cuda.synchronize()
    mem = buf.cpu().numpy()
    for t, (x, o) in enumerate(zip(xs, offs)):
        ref, s = O.encode(x.cpu().numpy(), "dynamic-tree", "absmax")
        got = mem[o:o + x.numel()]
        sc = float(np.frombuffer(mem[L + 4 * t:L + 4 * t + 4].tobytes(), np.float32)[0])
        assert sc == s, (t, sc, s)
        assert np.array_equal(got, ref), (t, int((got != ref).sum()))


def test_calls_with_different_segment_counts_share_a_workspace(cuda):
    """Regression: the workspace layout must not depend on a call's segment
    count (a 1-segment call once overwrote a 7-segment call's control slots)."""
    rng = np.random.default_rng(6)
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    for sizes in ([5000], [1200, 1, 17, 300, 64, 5000, 12544], [70000], [3, 9000, 40, 12544, 1, 2, 7, 100],
                  [1], [1200, 1, 17, 300, 64, 5000, 12544]):
        xs = [(rng.normal(size=n) * 1e-2).astype(np.float32) for n in sizes]
        check(xs, spec, cuda)


def test_resident_and_ticket_encoders_interleave(cuda):
    """Calls that fit in shared memory take the resident single-pass kernel,
    larger ones the ticket kernel; both share one workspace on the stream and
    must leave it as the other expects (alternating calls, all bit-exact)."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    rng = np.random.default_rng(77)
    small = [rng.normal(0, 0.1, size=n).astype(np.float32) for n in (3000, 1, 70001, 5)]
    large = [rng.normal(0, 0.01, size=n).astype(np.float32) for n in (8_000_003, 4097)]
    for xs in (small, large, small, large, small):
        check(xs, spec, cuda)


@pytest.mark.parametrize("sizes", [
    [(1,)], [(3,)], [(4096,)], [(7,), (0,), (9,)], [(51195,)], [(51196,)], [(51197,)],
    [(7_500_000,)], [(1_000_001,), (17,), (0,), (3_000_000,)],
    [(int(n),) for n in np.random.default_rng(3).integers(0, 20000, size=32)],
])
def test_resident_sizes(cuda, sizes):
    """Piece boundaries of the resident kernel: single elements, ragged ends,
    empty segments, per-CTA capacity edges (51196 = 200 KB / 4 - 4) and the
    largest call that still fits."""
    spec = A.DataTypeSpec("linear", "absmax")
    rng = np.random.default_rng(len(sizes))
    xs = [rng.normal(0, 1.0, size=s).astype(np.float32) for s in sizes]
    check(xs, spec, cuda)
    if len(xs) > 1:
        check(xs, spec, cuda, nblocks=3)  # two_round-style multi-block layout
