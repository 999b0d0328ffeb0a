"""GPU error bench (approx8/errorbench.py) and hook statistics (mlp.py:146-164).

CPU tests pin the oracle restatement and the host-side API (validation,
labels, suite layout, CSV/table rendering) to reference outputs in
tests/golden/errorbench.json (made by tests/golden/make_golden_errorbench.py
from the real reference).  GPU tests run the sm_100a round trip + the fused
error-sum kernel (a8_error_stats) and compare with the goldens: the per-
element arithmetic is the reference's, the float64 sums differ only in
summation order, so aggregates are compared at rel 1e-12 (the reference's
own tolerance, test_errorbench.py:76-77) and the rendered CSV must be equal.
"""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

import paper_1511_04561_b200 as A
from paper_1511_04561_b200 import errorbench as EB
from helpers import GOLDEN, parse_tag
from oracle import approx8_oracle as O

G = json.loads((GOLDEN / "errorbench.json").read_text())
REL = 1e-12


def cell_inputs():
    """Same recipes as tests/golden/make_golden_errorbench.py:cell_inputs."""
    rng = np.random.default_rng(11)
    yield "rescan_normal1000", rng.normal(size=1000).astype(np.float32)
    rng = np.random.default_rng(12)
    yield "normal4096_x1024", (rng.normal(size=4096).astype(np.float32) * np.float32(1024.0))
    rng = np.random.default_rng(13)
    x = rng.normal(0, 0.01, size=100_003)
    x[::7] = 0.0
    yield "f64_zeros", x
    yield "single", np.array([0.3], dtype=np.float32)
    yield "allzero", np.zeros(257, dtype=np.float32)
    rng = np.random.default_rng(14)
    yield "uniform_1e6", rng.random(1_000_000).astype(np.float32)


def spec_of(label: str) -> A.DataTypeSpec:
    return A.parse_spec(label)


def reports_from(golden_reports):
    return [EB.ErrorReport(spec=spec_of(r["spec"]), mean_abs_error=r["mean_abs_error"],
                           mean_rel_error_pct=r["mean_rel_error_pct"], count=r["n"],
                           sample_label=r["dist"], seed=r["seed"]) for r in golden_reports]


# ---------------------------------------------------------------------------
# CPU: oracle and host logic


def test_oracle_measure_error_matches_reference_cells():
    inputs = dict(cell_inputs())
    for c in G["cells"]:
        kind, norm, dec = parse_tag(c["spec"])
        m, r, n = O.measure_error(inputs[c["input"]], kind, norm, dec)
        assert (m, r, n) == (c["mean_abs_error"], c["mean_rel_error_pct"], c["count"]), c


def test_oracle_error_sums_decompose_measure_error():
    x = dict(cell_inputs())["rescan_normal1000"]
    y = O.roundtrip(x, "dynamic-tree", "absmax")
    a, r, nz = O.error_sums(x, y)
    m, rel, n = O.measure_error(x, "dynamic-tree", "absmax")
    assert a / n == pytest.approx(m, rel=1e-15)
    assert 100 * r / nz == pytest.approx(rel, rel=1e-14)


def test_reports_to_csv_and_table_match_reference_text():
    reps = reports_from(G["suite_seed0"]["reports"])
    assert EB.reports_to_csv(reps) == G["suite_seed0"]["csv"]
    assert EB.format_table(reps) == G["suite_seed0"]["table"]
    assert EB.CSV_HEADER == ("distribution", "datatype", "n", "mean_abs_error", "mean_rel_error_pct", "seed")


def test_sample_matches_oracle_sampler():
    s = EB.SampleSpec(EB.DIST_NORMAL, 1000, seed=7, sigma=0.2)
    assert np.array_equal(EB.sample(s), O.sample_normal(1000, 7, 0.0, 0.2))
    u = EB.SampleSpec(EB.DIST_UNIFORM01, 1000, seed=3)
    assert np.array_equal(EB.sample(u), O.sample_uniform01(1000, 3))
    assert EB.sample(s).dtype == np.float32


def test_sample_spec_validation_and_labels():
    with pytest.raises(A.ConfigError):
        EB.SampleSpec("poisson", 10, seed=0)
    with pytest.raises(A.ConfigError):
        EB.SampleSpec(EB.DIST_NORMAL, 0, seed=0)
    with pytest.raises(A.ConfigError):
        EB.SampleSpec(EB.DIST_NORMAL, 10, seed=0, sigma=-1.0)
    assert EB.SampleSpec(EB.DIST_UNIFORM01, 1, 0).label() == "U(0,1)"
    assert EB.SampleSpec(EB.DIST_NORMAL, 1, 0, sigma=10.0).label() == "N(0,10^2)"
    assert EB.SampleSpec(EB.DIST_NORMAL, 1, 0, sigma=0.2).label() == "N(0,0.2^2)"


def test_suite_spec_protocol():
    K = A.DataTypeKind
    assert EB.suite_spec(K.DYNAMIC_TREE, EB.DIST_UNIFORM01, {}) == A.DataTypeSpec(K.DYNAMIC_TREE, A.NormKind.ABSMAX)
    assert EB.suite_spec(K.LINEAR, EB.DIST_NORMAL, {"sigma": 10.0}) == A.DataTypeSpec(K.LINEAR, A.NormKind.ABSMAX)
    assert EB.suite_spec(K.MANTISSA, EB.DIST_NORMAL, {"sigma": 10.0}) == A.DataTypeSpec(K.MANTISSA, A.NormKind.DECADE, 2)
    assert EB.suite_spec(K.STATIC_TREE, EB.DIST_NORMAL, {"sigma": 1.0}) == A.DataTypeSpec(K.STATIC_TREE, A.NormKind.DECADE, 1)
    labels = [(r["dist"], r["spec"]) for r in G["suite_seed0"]["reports"]]
    mine = []
    for dist, params in EB.SUITE_DISTRIBUTIONS:
        for kind in EB.SUITE_KINDS:
            mine.append((EB.SampleSpec(dist, 1, 0, **params).label(), EB.suite_spec(kind, dist, params).label()))
    assert mine == labels


def test_worker_count(monkeypatch):
    monkeypatch.setenv("APPROX8_THREADS", "3")
    assert EB.worker_count(16) == 3
    assert EB.worker_count(2) == 2
    monkeypatch.setenv("APPROX8_THREADS", "zero")
    with pytest.raises(A.ConfigError):
        EB.worker_count(4)


def test_error_stats_symbols_exported():
    from paper_1511_04561_b200 import _native as N

    assert N.lib.a8_error_workspace_bytes() > 0
    assert callable(N.lib.a8_error_stats)


# ---------------------------------------------------------------------------
# GPU: the sm_100a round trip + fused error sums


@pytest.mark.gpu
def test_measure_error_cells_match_reference(cuda):
    inputs = dict(cell_inputs())
    for c in G["cells"]:
        r = EB.measure_error(inputs[c["input"]], spec_of(c["spec"]), device=cuda)
        assert r.count == c["count"]
        assert r.mean_abs_error == pytest.approx(c["mean_abs_error"], rel=REL, abs=0.0), c
        assert r.mean_rel_error_pct == pytest.approx(c["mean_rel_error_pct"], rel=REL, abs=0.0), c


@pytest.mark.gpu
def test_run_error_suite_matches_reference(cuda):
    for key, seed, count in (("suite_seed0", 0, 1_000_000), ("suite_seed5", 5, 20_000)):
        reps = EB.run_error_suite(seed=seed, count=count, device=cuda)
        want = G[key]["reports"]
        assert len(reps) == 16
        for r, w in zip(reps, want):
            assert (r.sample_label, r.spec.label(), r.count, r.seed) == (w["dist"], w["spec"], w["n"], w["seed"])
            assert r.mean_abs_error == pytest.approx(w["mean_abs_error"], rel=REL, abs=0.0)
            assert r.mean_rel_error_pct == pytest.approx(w["mean_rel_error_pct"], rel=REL, abs=0.0)
        assert EB.reports_to_csv(reps) == G[key]["csv"]
    again = EB.run_error_suite(seed=5, count=20_000, device=cuda)
    assert again == EB.run_error_suite(seed=5, count=20_000, device=cuda)  # deterministic


@pytest.mark.gpu
def test_measure_error_codebook_values_are_exact(cuda):
    for kind in A.DataTypeKind:
        spec = A.DataTypeSpec(kind)
        values = A.build_codebook(spec).decode_table.astype(np.float32)
        r = EB.measure_error(values, spec, device=cuda)
        assert r.mean_abs_error == 0.0 and r.mean_rel_error_pct == 0.0, kind


@pytest.mark.gpu
def test_measure_error_errors(cuda):
    with pytest.raises(A.UsageError):
        EB.measure_error(np.empty(0, np.float32), A.DataTypeSpec("linear"), device=cuda)
    x = np.ones(100, np.float32)
    x[17] = np.nan
    with pytest.raises(A.InputError):
        EB.measure_error(x, A.DataTypeSpec("dynamic-tree", "absmax"), device=cuda)


@pytest.mark.gpu
def test_relative_error_scale_invariance_absmax(cuda):
    """test_errorbench.py:107-117: power-of-two factors cannot move codes."""
    x = np.random.default_rng(12).normal(size=4096).astype(np.float32)
    for kind in ("dynamic-tree", "linear"):
        spec = A.DataTypeSpec(kind, "absmax")
        base = EB.measure_error(x, spec, device=cuda)
        for c in (0.25, 2.0, 1024.0):
            assert EB.measure_error(x * np.float32(c), spec, device=cuda).mean_rel_error_pct == base.mean_rel_error_pct


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3, 4097, 1 << 22])
def test_error_sums_vs_oracle_sizes(cuda, n):
    """Ragged and large sizes, unaligned tails, torch input on the device."""
    x = O.sample_normal(n, 100 + n, 0.0, 0.05)
    x[::5] = 0.0
    for tag in ("dynamic-tree/absmax", "static-tree/decade+1"):
        kind, norm, dec = parse_tag(tag)
        want = O.measure_error(x, kind, norm, dec)
        r = EB.measure_error(torch.from_numpy(x).to(cuda), A.parse_spec(tag))
        assert r.count == want[2]
        assert r.mean_abs_error == pytest.approx(want[0], rel=REL, abs=0.0)
        assert r.mean_rel_error_pct == pytest.approx(want[1], rel=REL, abs=0.0)


@pytest.mark.gpu
def test_hook_stats_record_and_codes_agree_with_reference_formula(cuda):
    """mlp.py:146-164: record(before, after) and the fused record_codes give
    the reference sums; summary() = (abs_sum/n, 100*rel_sum/nnz) per layer."""
    spec = A.DataTypeSpec("dynamic-tree", "absmax")
    cb = A.build_codebook(spec)
    stats_a, stats_b = A.HookStats(), A.HookStats()
    tot = {}
    for layer, (n, seed) in enumerate([(5000, 1), (128 * 512, 2), (77, 3)]):
        for step in range(3):
            x = O.sample_normal(n, seed * 10 + step, 0.0, 0.1)
            x[::3] = 0.0
            y = O.roundtrip(x, "dynamic-tree", "absmax")
            xt = torch.from_numpy(x).to(cuda)
            stats_a.record("forward", layer, xt, torch.from_numpy(y).to(cuda))
            stats_b.record_codes("forward", layer, xt, A.encode_buffer(xt, cb), cb)
            a, r, nz = O.error_sums(x, y)
            acc = tot.setdefault(layer, [0.0, 0.0, 0, 0])
            acc[0] += a
            acc[1] += r
            acc[2] += n
            acc[3] += nz
    sa, sb = stats_a.summary()["forward"], stats_b.summary()["forward"]
    assert sa == sb
    for layer, (a, r, n, nz) in tot.items():
        assert sa[layer][0] == pytest.approx(a / n, rel=REL, abs=0.0)
        assert sa[layer][1] == pytest.approx(100.0 * r / nz, rel=REL, abs=0.0)


@pytest.mark.gpu
def test_make_quantizer_records_fused_stats(cuda):
    spec = A.default_hook_spec("mantissa", "model-parallel")
    stats = A.HookStats()
    qz = A.make_quantizer(spec, stats, "backward")
    x64 = np.random.default_rng(4).normal(0, 0.02, size=(128, 512))
    y = qz(torch.from_numpy(x64).to(cuda), 2)
    want = O.roundtrip(x64, "mantissa", "decade", 2)
    assert y.dtype == torch.float64
    assert np.array_equal(y.cpu().numpy(), want.astype(np.float64))
    a, r, nz = O.error_sums(x64, want)
    got = stats.summary()["backward"][0]
    assert got[0] == pytest.approx(a / x64.size, rel=REL, abs=0.0)
    assert got[1] == pytest.approx(100.0 * r / nz, rel=REL, abs=0.0)


@pytest.mark.gpu
def test_cli_bench_error_matches_reference_csv(cuda, tmp_path):
    """`python -m paper_1511_04561_b200.errorbench` mirrors the reference CLI's
    bench-error (cli.py:119-125): same CSV text for the same seed and count."""
    out = tmp_path / "suite.csv"
    assert EB.main(["--n", "20000", "--seed", "5", "--out", str(out)]) == 0
    assert out.read_text() == G["suite_seed5"]["csv"]
    tab = tmp_path / "suite.txt"
    assert EB.main(["--n", "20000", "--seed", "5", "--table", "--out", str(tab)]) == 0
    assert tab.read_text().splitlines()[0].startswith("distribution")
