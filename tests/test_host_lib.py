"""CPU tests of the product library's host side and Python API surface.

No compute kernel runs here (no GPU): these check that the C-ABI library
loads and exports every symbol include/approx8_b200.h declares, that its host
builders (codebooks, fixed scales, decision tables) are bit-exact against the
reference goldens, and that the API mirrors the reference's validation and
error taxonomy.  The compute path itself has no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import io
import re

import numpy as np
import pytest
import torch

from helpers import ROOT, O, golden, golden_cases

import paper_1511_04561_b200 as A
from paper_1511_04561_b200 import _native as N
from paper_1511_04561_b200.exchange import make_plan


def header_functions():
    text = (ROOT / "include" / "approx8_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+)+\**(a8_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 9
    for name in names:
        assert hasattr(N.lib, name), name
        assert name in N.SIGNATURES, name
    assert N.lib.a8_abi_version() == 1


def test_struct_sizes_match_the_header():
    assert C.sizeof(N.Book) == 1024 + 1024 + 128 + 16
    assert C.sizeof(N.Lut) == 32 + 512 + 4 * N.LUT_MAX
    assert C.sizeof(N.EncSeg) == 32 and C.sizeof(N.DecSeg) == 32
    assert C.sizeof(N.Layout) == 56
    assert C.sizeof(N.ObSeg) == 24
    assert C.sizeof(N.ProdSeg) == 32


@pytest.mark.parametrize("kind", ["dynamic-tree", "static-tree", "linear", "mantissa"])
def test_codebook_matches_reference(kind):
    g, meta = golden()
    cb = A.build_codebook(A.DataTypeSpec(kind))
    assert cb.decode_table.tobytes() == g[f"table/{kind}"].tobytes()
    assert np.array_equal(cb.sorted_values, g[f"values/{kind}"])
    assert np.array_equal(cb.sorted_codes, g[f"codes/{kind}"])
    assert cb.zero_code == 0
    with pytest.raises(ValueError):
        cb.decode_table[0] = 1.0
    assert A.build_codebook(A.DataTypeSpec(kind)) is cb


def test_codebook_dump_format():
    cb = A.build_codebook(A.DataTypeSpec("mantissa"))
    buf = io.StringIO()
    cb.dump(buf)
    lines = buf.getvalue().splitlines()
    assert len(lines) == 256 and lines[0] == "0x00\t0"
    assert lines[0x12] == f"0x12\t{np.float32(0.2):.9g}"


def test_spec_validation_matrix():
    A.DataTypeSpec(A.DataTypeKind.DYNAMIC_TREE, A.NormKind.ABSMAX)
    A.DataTypeSpec(A.DataTypeKind.STATIC_TREE, A.NormKind.DECADE, -3)
    for bad in [("dynamic-tree", "decade", 1), ("mantissa", "absmax", 0),
                ("static-tree", "decade", 8), ("linear", "none", 2), ("bogus", "none", 0)]:
        with pytest.raises(A.ConfigError):
            A.DataTypeSpec(*bad)
    s = A.DataTypeSpec("mantissa", "decade", 2)
    assert s.label() == "mantissa/decade+2"
    assert A.parse_spec(s.label()) == s
    assert A.parse_spec("linear/absmax") == A.DataTypeSpec("linear", "absmax")


@pytest.mark.parametrize("dec", range(-7, 8))
def test_fixed_scales_match_reference(dec):
    cb = A.build_codebook(A.DataTypeSpec("static-tree", "decade", dec))
    assert cb.fixed_scale == O.scale_of(np.zeros(1), "decade", dec)
    assert A.build_codebook(A.DataTypeSpec("linear")).fixed_scale == 1.0
    assert A.build_codebook(A.DataTypeSpec("linear", "absmax")).fixed_scale is None


def _lut_encode(x, lut, book):
    """NumPy restatement of a8_core.cuh encode_lut/encode_search over a host-built table."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    a = b & np.uint32(0x7FFFFFFF)
    if lut.valid:
        e = np.frombuffer(bytes(lut.e), np.uint32)
        j = np.clip((a >> 16).astype(np.int64) - lut.kbase, 0, lut.len - 1)
        v = e[j]
        c = np.where(((a << 16) | 0xFFFF) >= v, v >> 8, v) & 0xFF
    else:
        T = np.frombuffer(bytes(lut.T), np.uint32)[:127]
        c = np.frombuffer(bytes(book.codes), np.uint8)[np.searchsorted(T, a, side="right")].astype(np.uint32)
    return (c | ((c + 0x7F) & (b >> 24) & 0x80)).astype(np.uint8)


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0])
def test_host_decision_table_reproduces_reference(case):
    name, spec, x, ref = case
    s = O.encode(x, *spec)[1]
    cb = A.build_codebook(A.DataTypeSpec(spec[0]))
    lut = N.Lut()
    N.check(N.lib.a8_build_lut_host(C.byref(cb._book), s, C.byref(lut)))
    T = np.frombuffer(bytes(lut.T), np.uint32)[:127]
    assert np.array_equal(T, O.thresholds(spec[0], s)), name
    assert np.array_equal(_lut_encode(x, lut, cb._book), ref), name
    if s >= 1e-30:
        assert lut.valid == 1 and lut.len <= N.LUT_MAX, name


def _carry_table(T, amax_bits):
    """NumPy restatement of the device's carry-table build (a8_kernels.cu
    fill_lut_local<true> + the absmax length extension, a8_core.cuh
    carry_entry): returns (entries, kbase) or None when a bucket would hold
    two thresholds (the kernel then searches the thresholds)."""
    F = int(np.count_nonzero(T < 0x7F800000))
    if F == 0:
        kbase, length = 0, 1
    else:
        kbase = int(T[0] >> 16) - 1
        length = int(T[F - 1] >> 16) - int(T[0] >> 16) + 3
    length = max(length, int(amax_bits >> 16) - kbase + 1)
    if length > N.LUT_MAX:
        return None
    keys = np.arange(length, dtype=np.int64) + kbase
    tk = (T[:F] >> 16).astype(np.int64)
    lo = np.searchsorted(tk, keys, side="left")
    cnt = np.searchsorted(tk, keys, side="right") - lo
    if cnt.max(initial=0) > 1:
        return None
    tl = np.where(cnt > 0, T[np.minimum(lo, 126)] & 0xFFFF, 0).astype(np.int64)
    e = ((lo << 16) + np.where(cnt > 0, 0x10000 - tl, 0)).astype(np.uint32)
    return e, kbase


def _carry_encode(x, e, kbase):
    """The device formula of carry_sum / pack4_carry, element-wise: index
    max(key - kbase, 0) with NO upper clamp (it must stay in the table),
    code = byte 2 of e + (b & 0x8000ffff), sign from byte 3."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    j = np.maximum(((b & 0x7FFF0000) >> 16).astype(np.int64) - kbase, 0)
    assert j.max(initial=0) < e.size, "an element indexes past the table"
    ssum = (e[j].astype(np.uint64) + (b & 0x8000FFFF)) & 0xFFFFFFFF
    c = (ssum >> 16) & 0xFF
    sign = (ssum >> 24) & 0xFF
    assert np.all((sign == 0) | (sign == 0x80)) and np.all(c < 128)
    return (c | (sign & ((c + 0x7F) & 0x80))).astype(np.uint8)


@pytest.mark.parametrize("case", [c for c in golden_cases() if c[1][1] == "absmax"], ids=lambda c: c[0])
def test_carry_table_reproduces_reference(case):
    """The absmax encode kernel's carry table (monotone codebooks), restated
    on the host with its exact integer arithmetic, gives the reference codes."""
    name, spec, x, ref = case
    assert spec[0] in ("dynamic-tree", "linear")
    assert np.array_equal(O.book(spec[0]).codes, np.arange(128, dtype=np.uint8))  # canonical code == index
    s = O.encode(x, *spec)[1]
    cb = A.build_codebook(A.DataTypeSpec(spec[0]))
    lut = N.Lut()
    N.check(N.lib.a8_build_lut_host(C.byref(cb._book), s, C.byref(lut)))
    T = np.frombuffer(bytes(lut.T), np.uint32)[:127]
    amax = int(np.abs(np.asarray(x, np.float32)).view(np.uint32).max(initial=0)) if x.size else 0
    built = _carry_table(T, amax)
    if built is None:  # the kernel searches the thresholds instead
        assert s < 1e-30, name
        return
    assert np.array_equal(_carry_encode(x, *built), ref), name


def test_error_codes_map_to_reference_exceptions():
    with pytest.raises(A.ConfigError):
        N.check(N.lib.a8_codebook(9, C.byref(N.Book())))
    s = C.c_float()
    with pytest.raises(A.ConfigError):
        N.check(N.lib.a8_fixed_scale(2, 9, C.byref(s)))
    with pytest.raises(A.UsageError):
        N.check(N.lib.a8_fixed_scale(1, 0, C.byref(s)))
    lay = N.Layout()
    with pytest.raises(A.UsageError):  # no segment: rejected before any launch
        N.check(N.lib.a8_encode(None, 0, None, 1, None, lay, None, 0, None, None, None))
    with pytest.raises(A.UsageError):
        N.check(N.lib.a8_decode((N.DecSeg * 1)(), 1, C.c_void_p(16), lay, 0, 0, -1, 0, None,
                                C.c_void_p(16), 0, None))


def test_compute_has_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present; covered by -m gpu")
    cb = A.build_codebook(A.DataTypeSpec("linear", "absmax"))
    with pytest.raises(Exception):
        A.encode_buffer(np.ones(8, np.float32), cb)
    with pytest.raises(Exception):
        A.roundtrip(np.ones(8, np.float32), cb.spec)


def test_decode_usage_errors_before_any_device_work():
    cb_lin = A.build_codebook(A.DataTypeSpec("linear"))
    cb_dyn = A.build_codebook(A.DataTypeSpec("dynamic-tree"))
    q = A.QuantizedTensor(np.zeros(4, np.uint8), (4,), cb_lin.spec, 1.0)
    with pytest.raises(A.UsageError):
        A.decode_buffer(q, cb_dyn)
    q1 = A.QuantizedTensor(np.zeros(1, np.uint8), (4,), None, 1.0, nbits=1)
    with pytest.raises(A.UsageError):
        A.decode_buffer(q1, cb_lin)


@pytest.mark.parametrize("nranks", [1, 2, 3, 8])
def test_exchange_plan_layout(nranks):
    sizes = [0, 1, 15, 16, 17, 4096, 12345, 7]
    p = make_plan(sizes, nranks)
    assert all(o % 16 == 0 for o in p.offs)
    assert p.shard % 16 == 0 and p.shard * nranks >= p.offs[-1] + sizes[-1]
    assert p.gap % 16 == 0 and p.gap >= 4 * (len(sizes) + 1)
    cover = {}
    for pc in p.pieces:
        assert pc.flat // p.shard == pc.shard
        assert (pc.flat + pc.n - 1) // p.shard == pc.shard
        assert pc.flat % 16 == 0 and pc.start % 16 == 0
        cover[pc.tensor] = cover.get(pc.tensor, 0) + pc.n
    assert all(cover.get(t, 0) == n for t, n in enumerate(sizes))
    per = {}
    for pc in p.pieces:
        per.setdefault(pc.shard, []).append(pc.idx)
    for idxs in per.values():
        assert idxs == list(range(len(idxs))) and len(idxs) <= len(sizes)


def test_hook_config_mirrors_reference():
    with pytest.raises(A.ConfigError):
        A.QuantHookConfig(A.HookMode.MODEL_PARALLEL, "onebit")
    with pytest.raises(A.ConfigError):
        A.QuantHookConfig(A.HookMode.DATA_PARALLEL, "twobit")
    assert not A.QuantHookConfig().active
    assert A.QuantHookConfig(A.HookMode.DATA_PARALLEL, A.DataTypeSpec("linear")).label() == "linear/none [data-parallel]"
    assert A.default_hook_spec("dynamic-tree", "model-parallel") == A.DataTypeSpec("dynamic-tree", "absmax")
    assert A.default_hook_spec("mantissa", "model-parallel") == A.DataTypeSpec("mantissa", "decade", 2)
    assert A.default_hook_spec("static-tree", "data-parallel") == A.DataTypeSpec("static-tree")


@pytest.mark.parametrize("kind", ["dynamic-tree", "static-tree", "linear", "mantissa"])
def test_thresholds_at_random_scales_match_bisection(kind):
    """The library's guess-and-walk threshold search equals the oracle's full
    bisection of the reference decision at random and extreme scales."""
    rng = np.random.default_rng({"dynamic-tree": 1, "static-tree": 2, "linear": 3, "mantissa": 4}[kind])
    scales = list((10.0 ** rng.uniform(-44, 38, size=12)).astype(np.float32))
    scales += [np.float32(x) for x in (1e-45, 2.5e-42, 1.1754942e-38, 1.0, 3.4028235e38, 4.998160362243652)]
    cb = A.build_codebook(A.DataTypeSpec(kind))
    for s in scales:
        if not np.isfinite(s) or s <= 0:
            continue
        lut = N.Lut()
        N.check(N.lib.a8_build_lut_host(C.byref(cb._book), float(s), C.byref(lut)))
        T = np.frombuffer(bytes(lut.T), np.uint32)[:127]
        assert np.array_equal(T, O.thresholds(kind, float(s))), (kind, s)


def test_parallel_threshold_window(tmp_path):
    """The resident kernel tests the 8 float32 patterns around the rounded
    midpoint in parallel (threshold_parallel); on the host, over random
    normal scales and all four codebooks, that window must give exactly
    threshold()'s result (or fall back to it)."""
    import shutil
    import subprocess

    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    root = ROOT
    exe = tmp_path / "threshold_window"
    subprocess.run([gxx, "-O2", "-std=c++17", f"-I{root / 'paper_1511_04561_b200' / 'csrc'}", f"-I{root / 'include'}",
                    str(root / "tests" / "cpp" / "threshold_window.cpp"),
                    str(root / "paper_1511_04561_b200" / "csrc" / "a8_codebook.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "1500"], capture_output=True, text=True)
    total, bad, fallback, bad_fast = (int(v) for v in out.stdout.split())
    assert out.returncode == 0 and bad == 0 and bad_fast == 0, out.stdout
    assert total > 700_000 and fallback < total // 50
