"""The oracle is pinned to the REAL reference before it is trusted (CPU).

Golden vectors come from tests/golden/make_golden.py, which imports the
reference package in the build container.  Every check here is bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import O, acceptance_inputs, fullrange_cases, golden, golden_cases, sha, tag

KINDS = ("dynamic-tree", "static-tree", "linear", "mantissa")


@pytest.mark.parametrize("kind", KINDS)
def test_tables_match_reference(kind):
    g, meta = golden()
    bk = O.book(kind)
    assert bk.table.tobytes() == g[f"table/{kind}"].tobytes()
    assert np.array_equal(bk.values, g[f"values/{kind}"])
    assert np.array_equal(bk.codes, g[f"codes/{kind}"])
    assert sha(bk.table) == meta["tables"][kind]["sha_table"]
    assert len(bk.values) == meta["tables"][kind]["ndistinct"]


def test_table_digests_are_the_published_pins():
    # BASELINE.md §4
    pins = {"dynamic-tree": "d99d3890d8b1e964", "static-tree": "6fda742767a44a70",
            "linear": "b55cb6713a2220ee", "mantissa": "d6e6312451c11fee"}
    for kind, d in pins.items():
        assert sha(O.book(kind).table) == d


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0])
def test_encode_matches_reference_vectors(case):
    name, spec, x, ref = case
    codes, s = O.encode(x, *spec)
    assert np.array_equal(codes, ref), name
    # and the reference's independent exhaustive scan (oracles.py:24-45); it
    # is only meaningful where |x|/s is moderate (for |y| ~ 1e38 every fp64
    # distance rounds to the same value and its tie rule picks 0), which is
    # the domain the reference tests use it on (|x| <= 1e3)
    y = np.abs(x.astype(np.float64)) / s
    keep = y <= 1e6
    if keep.all():
        assert np.array_equal(O.exhaustive_codes(x, *spec), ref), name
    else:  # fixed-scale specs only (absmax keeps |y| <= 1)
        assert spec[1] != "absmax"
        assert np.array_equal(O.exhaustive_codes(x[keep], *spec), ref[keep]), name
    # and the threshold reformulation the kernels use
    assert np.array_equal(O.encode_by_thresholds(x, spec[0], s), ref), name


def test_fullrange_buffers_match_reference():
    for base, spec, xs, cs, scales in fullrange_cases():
        for x, c, s in zip(xs, cs, scales):
            got, gs = O.encode(x, *spec)
            assert np.array_equal(got, c), base
            assert gs == s, base


def test_acceptance_digests():
    _, meta = golden()
    for spec, x in acceptance_inputs():
        m = meta["acceptance"][tag(spec)]
        assert sha(x) == m["sha_x"]
        codes, s = O.encode(x, *spec)
        assert sha(codes) == m["sha_codes"], tag(spec)
        assert sha(O.decode(codes, s, spec[0])) == m["sha_decoded"], tag(spec)
        assert s == m["scale"]


def test_config1_digests():
    _, meta = golden()
    x = O.sample_normal(2**20, 0)
    assert sha(x) == meta["c1"]["sha_x"]
    for t, m in meta["c1"].items():
        if t == "sha_x":
            continue
        kind, norm = t.split("/")
        dec = int(norm[6:]) if norm.startswith("decade") else 0
        norm = "decade" if norm.startswith("decade") else norm
        codes, s = O.encode(x, kind, norm, dec)
        assert sha(codes) == m["sha_codes"], t
        assert sha(O.decode(codes, s, kind)) == m["sha_decoded"], t
        assert s == m["scale"]


def test_error_suite_cells_match_reference():
    """run_error_suite(seed=0, count=1e6): bit-exact codes => identical stats."""
    _, meta = golden()
    dists = [("uniform01", {}), ("normal", {"sigma": 1.0}), ("normal", {"sigma": 10.0}),
             ("normal", {"sigma": 0.2})]
    kinds = ["dynamic-tree", "linear", "mantissa", "static-tree"]
    cells = meta["suite"]
    i = 0
    for d_idx, (dist, par) in enumerate(dists):
        for k_idx, kind in enumerate(kinds):
            seed = d_idx * 4 + k_idx
            x = (O.sample_uniform01(1_000_000, seed) if dist == "uniform01"
                 else O.sample_normal(1_000_000, seed, 0.0, par["sigma"]))
            if kind in ("dynamic-tree", "linear"):
                spec = (kind, "absmax", 0)
            else:
                spec = (kind, "decade", 2 if par.get("sigma", 1.0) >= 10 else 1)
            y = O.roundtrip(x, *spec)
            x64, y64 = x.astype(np.float64), y.astype(np.float64)
            err = np.abs(x64 - y64)
            nz = x64 != 0
            rel = float(np.mean(err[nz] / np.abs(x64[nz])) * 100.0)
            assert cells[i]["seed"] == seed
            assert float(err.mean()) == cells[i]["mean_abs_error"]
            assert rel == cells[i]["mean_rel_error_pct"]
            i += 1


def test_exchange_oracle_degenerates_to_roundtrip():
    rng = np.random.default_rng(5)
    g = [rng.normal(size=(33, 7)).astype(np.float32), rng.normal(size=5).astype(np.float32)]
    for fn in (O.exchange_allgather, O.exchange_two_round):
        out = fn([g], "dynamic-tree", "absmax")
        for a, b in zip(out, g):
            assert np.array_equal(a, O.roundtrip(b, "dynamic-tree", "absmax"))


def test_two_round_pieces_cover_every_element():
    offs, L = O.shard_bounds([5, 100, 17, 3], 3)
    assert all(o % 16 == 0 for o in offs) and L % 16 == 0
    assert L * 3 >= offs[-1] + 3


def test_c_restatement_matches_reference_vectors():
    for name, spec, x, ref in golden_cases():
        codes, s = O.c_encode(x, *spec)
        assert np.array_equal(codes, ref), name
        assert s == O.encode(x, *spec)[1]
        assert O.c_decode(ref, s, spec[0]).tobytes() == O.decode(ref, s, spec[0]).tobytes()
    _, meta = golden()
    x = O.sample_normal(2**20, 0)
    codes, s = O.c_encode(x, "dynamic-tree", "absmax")
    assert sha(codes) == meta["c1"]["dynamic-tree/absmax"]["sha_codes"]
    with pytest.raises(O.NonFinite):
        O.c_encode(np.array([1.0, np.nan], np.float32), "linear")


def test_onebit_restatement_matches_reference_chain():
    """oracle.onebit_quantize / onebit_decode (codecs.py:306-348) against the
    12 chained steps the real reference produced (residual carried)."""
    g, _ = golden()
    res = np.zeros(3000)
    for k in range(12):
        bits, pos, neg, res = O.onebit_quantize(g[f"onebit/{k}/g"], res)
        assert np.array_equal(bits, g[f"onebit/{k}/bits"]), k
        assert (pos, neg) == tuple(g[f"onebit/{k}/levels"]), k
        assert res.tobytes() == g[f"onebit/{k}/residual"].tobytes(), k
        assert O.onebit_decode(bits, 3000, pos, neg).tobytes() == g[f"onebit/{k}/decoded"].tobytes(), k
    # the exchange oracle at N = 1 is the chained quantize/decode itself
    r1 = [[np.zeros(3000)]]
    for k in range(3):
        out = O.exchange_onebit([[g[f"onebit/{k}/g"]]], r1)[0]
        assert out.tobytes() == g[f"onebit/{k}/decoded"].tobytes(), k
