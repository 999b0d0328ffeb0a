"""Generate golden vectors from the REAL reference (``approx8``) for parity pins.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz`` (arrays) and ``tests/golden/golden.json``
(digests, scales, error-suite cells).  Inputs that are large are not stored:
they are regenerated from the same seeded recipe in the tests and compared by
sha256 digest of the reference outputs.

Recipes (reference file:line they mirror):
  tables          codecs.py:186-204 (build_codebook) for the four kinds
  acceptance      test_acceptance.py:116-129, rng 20240818, 4 specs x 100k
  c1              errorbench.sample(normal, 2**20, seed 0) -- BASELINE config 1
  scan_<spec>     test_codecs.py:310-319 with a fixed seed per spec (the
                  reference seeds with hash(label), which is per-process)
  adversarial     threshold neighbours, exact midpoints, table values,
                  +-0, denormals, extreme magnitudes, per spec and scale
  extreme_absmax  absmax peaks from subnormal to FLT_MAX
  fullrange       finite float32 bit patterns in buffers of 1..24 elements
                  (the hypothesis domain of test_properties.py:47)
  suite           errorbench.run_error_suite(seed=0, count=1e6)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("APPROX8_REF", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))

from approx8 import codecs as C  # noqa: E402
from approx8 import errorbench as EB  # noqa: E402

OUT = Path(__file__).resolve().parent

SPECS = [
    ("dynamic-tree", "none", 0),
    ("dynamic-tree", "absmax", 0),
    ("linear", "none", 0),
    ("linear", "absmax", 0),
    ("static-tree", "none", 0),
    ("static-tree", "decade", 1),
    ("static-tree", "decade", -3),
    ("mantissa", "none", 0),
    ("mantissa", "decade", 2),
    ("mantissa", "decade", 1),
    ("mantissa", "decade", -1),
]


def dspec(kind, norm, dec):
    return C.DataTypeSpec(C.DataTypeKind(kind), C.NormKind(norm), dec)


def tag(kind, norm, dec):
    return f"{kind}/{norm}{dec:+d}" if norm == "decade" else f"{kind}/{norm}"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def ref_encode(x, spec):
    cb = C.build_codebook(dspec(*spec))
    q = C.encode_buffer(x, cb)
    return q.codes.copy(), float(q.scale), C.decode_buffer(q, cb).astype(np.float32).ravel()


def adversarial_inputs(kind, scale):
    """float32 values straddling every decision point of ``kind`` at ``scale``."""
    cb = C.build_codebook(C.DataTypeSpec(C.DataTypeKind(kind)))
    v = cb.sorted_values
    s = np.float64(np.float32(scale))
    pts = []
    mids = (v[:-1] + v[1:]) / 2.0 * s
    for m in mids:
        f = np.float32(m)
        b = np.array([f], np.float32).view(np.uint32)[0]
        for d in range(-3, 4):
            pts.append(np.uint32(max(0, int(b) + d)))
    tv = (v * s).astype(np.float32).view(np.uint32)
    for b in tv:
        for d in (-1, 0, 1):
            pts.append(np.uint32(max(0, int(b) + d)))
    extra = np.array([0.0, 1e-45, 3e-45, 1e-38, 1.17549435e-38, 1e-30, 1e-10,
                      0.5, 1.0, 15.0, 16.0, 1e10, 3.0e38, 3.4028235e38], np.float32)
    a = np.concatenate([np.array(pts, np.uint32).view(np.float32), extra])
    a = a[np.isfinite(a)]
    return np.concatenate([a, -a]).astype(np.float32)


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": str(REF), "numpy": np.__version__, "tables": {}, "c1": {},
                  "acceptance": {}, "scan": {}, "adversarial": {}, "extreme": {},
                  "fullrange": {}}

    # tables
    for kind in ("dynamic-tree", "static-tree", "linear", "mantissa"):
        cb = C.build_codebook(C.DataTypeSpec(C.DataTypeKind(kind)))
        arrays[f"table/{kind}"] = cb.decode_table.copy()
        arrays[f"values/{kind}"] = cb.sorted_values.copy()
        arrays[f"codes/{kind}"] = cb.sorted_codes.copy()
        meta["tables"][kind] = {"sha_table": sha(cb.decode_table), "ndistinct": int(len(cb.sorted_values))}

    # acceptance (test_acceptance.py:116-129): same rng stream, same spec order
    rng = np.random.default_rng(20240818)
    acc_specs = [("dynamic-tree", "absmax", 0), ("static-tree", "none", 0),
                 ("mantissa", "none", 0), ("linear", "absmax", 0)]
    for spec in acc_specs:
        mags = 10.0 ** rng.uniform(-8.0, 3.0, size=100_000)
        x = (mags * rng.choice([-1.0, 1.0], size=mags.size)).astype(np.float32)
        codes, s, dec = ref_encode(x, spec)
        meta["acceptance"][tag(*spec)] = {"sha_x": sha(x), "sha_codes": sha(codes),
                                          "sha_decoded": sha(dec), "scale": s}
        arrays[f"acceptance/{tag(*spec)}/codes_head"] = codes[:4096]

    # config 1: errorbench.sample(normal, 2**20, seed 0), suite normalisations
    x1 = EB.sample(EB.SampleSpec("normal", 2**20, seed=0, sigma=1.0))
    meta["c1"]["sha_x"] = sha(x1)
    for spec in [("dynamic-tree", "absmax", 0), ("linear", "absmax", 0),
                 ("static-tree", "decade", 1), ("mantissa", "decade", 1)]:
        codes, s, dec = ref_encode(x1, spec)
        meta["c1"][tag(*spec)] = {"sha_codes": sha(codes), "sha_decoded": sha(dec), "scale": s}

    # scan (test_codecs.py:310-319) with fixed seeds; stored in full
    for i, spec in enumerate(SPECS):
        r = np.random.default_rng(1000 + i)
        x = r.normal(size=4000) * 10.0 ** r.integers(-8, 3, size=4000)
        cb = C.build_codebook(dspec(*spec))
        salt = np.concatenate([cb.decode_table, [0.0], cb.sorted_values[:-1] * 1.0000001])
        x = np.concatenate([x, salt]).astype(np.float32)
        codes, s, dec = ref_encode(x, spec)
        arrays[f"scan/{tag(*spec)}/x"] = x
        arrays[f"scan/{tag(*spec)}/codes"] = codes
        meta["scan"][tag(*spec)] = {"scale": s}

    # adversarial: decision-point neighbours at several scales (none/decade
    # fix the scale; for absmax the peak element pins the scale)
    for spec in SPECS:
        kind, norm, dec = spec
        scales = [float(np.float32(10.0 ** dec))] if norm == "decade" else [1.0]
        if norm == "absmax":
            scales = [1.0, 4.998160362243652, 3.0e-3, 7.5e4, 1.0e-20]
        for j, s in enumerate(scales):
            a = adversarial_inputs(kind, s)
            if norm == "absmax":
                a = a[np.abs(a) <= np.float32(s)]
                a = np.concatenate([[np.float32(s)], a]).astype(np.float32)
            codes, sc, decd = ref_encode(a, spec)
            key = f"adv/{tag(*spec)}/{j}"
            arrays[key + "/x"] = a
            arrays[key + "/codes"] = codes
            meta["adversarial"][key] = {"scale": sc}

    # extreme absmax peaks (subnormal .. FLT_MAX)
    r = np.random.default_rng(77)
    for kind in ("dynamic-tree", "linear"):
        for j, peak in enumerate([1e-45, 3e-44, 1e-40, 1.17e-38, 1e-30, 1.0, 1e30, 3.4e38]):
            p = np.float32(peak)
            pb = int(np.array([p], np.float32).view(np.uint32)[0])
            if pb < 70000:
                bits = np.arange(0, pb + 1, dtype=np.uint32)
            else:
                bits = r.integers(0, pb + 1, size=20000, dtype=np.uint64).astype(np.uint32)
                bits = np.concatenate([bits, [pb]]).astype(np.uint32)
            x = bits.view(np.float32)
            x = np.where(r.random(x.size) < 0.5, -x, x).astype(np.float32)
            spec = (kind, "absmax", 0)
            codes, s, decd = ref_encode(x, spec)
            key = f"extreme/{kind}/{j}"
            arrays[key + "/x"] = x
            arrays[key + "/codes"] = codes
            meta["extreme"][key] = {"scale": s, "peak": float(p)}

    # full-range finite float32 buffers of 1..24 elements
    r = np.random.default_rng(99)
    for spec in SPECS:
        xs, cs, sizes, scs = [], [], [], []
        for _ in range(200):
            n = int(r.integers(1, 25))
            bits = r.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
            x = bits.view(np.float32)
            bad = ~np.isfinite(x)
            x[bad] = np.float32(0.0)
            codes, s, decd = ref_encode(x, spec)
            xs.append(x); cs.append(codes); sizes.append(n); scs.append(s)
        key = f"full/{tag(*spec)}"
        arrays[key + "/x"] = np.concatenate(xs)
        arrays[key + "/codes"] = np.concatenate(cs)
        arrays[key + "/sizes"] = np.array(sizes, np.int32)
        arrays[key + "/scales"] = np.array(scs, np.float64)

    # float64 inputs (the reference's DP/MP seams feed float64, mlp.py:330):
    # values float32 cannot represent, exact midpoints, wide magnitudes
    r = np.random.default_rng(51)
    for spec in SPECS:
        x = r.normal(size=3000) * 10.0 ** r.integers(-8, 3, size=3000)
        cb = C.build_codebook(dspec(*spec))
        mids = (cb.sorted_values[:-1] + cb.sorted_values[1:]) / 2.0
        x = np.concatenate([x, mids, -mids, mids * (1 + 2**-52), np.nextafter(mids, 0)])
        codes, s, _ = ref_encode(x, spec)
        arrays[f"f64/{tag(*spec)}/x"] = x
        arrays[f"f64/{tag(*spec)}/codes"] = codes
        meta.setdefault("f64", {})[tag(*spec)] = {"scale": s}

    # A8T1 files written by the reference (tensorfile.py:56-88): byte images
    import tempfile

    from approx8 import tensorfile as TF

    meta["a8t1"] = {}
    with tempfile.TemporaryDirectory() as td:
        def ref_file(obj, name):
            fp = Path(td) / name
            TF.write_tensor(fp, obj)
            return fp.read_bytes()

        x1 = EB.sample(EB.SampleSpec("normal", 2**20, seed=0, sigma=1.0))
        cb = C.build_codebook(dspec("dynamic-tree", "absmax", 0))
        meta["a8t1"]["c1_dynamic_absmax_sha"] = sha(np.frombuffer(ref_file(C.encode_buffer(x1, cb), "c1.a8t"), np.uint8))
        r = np.random.default_rng(31)
        small = (r.normal(size=(3, 4, 5)) * 0.1).astype(np.float32)
        arrays["a8t1/small_x"] = small
        for spec in [("dynamic-tree", "absmax", 0), ("mantissa", "decade", -2), ("linear", "none", 0)]:
            q = C.encode_buffer(small, C.build_codebook(dspec(*spec)))
            arrays[f"a8t1/codes/{tag(*spec)}"] = np.frombuffer(ref_file(q, "q.a8t"), np.uint8)
        arrays["a8t1/float32"] = np.frombuffer(ref_file(small, "f.a8t"), np.uint8)
        st = C.OneBitState.zeros(small.shape)
        qb = C.onebit_quantize(small.astype(np.float64), st)
        arrays["a8t1/onebit"] = np.frombuffer(ref_file(qb, "b.a8t"), np.uint8)

    # 1-bit error-feedback quantizer (codecs.py:291-348): 12 chained steps
    r = np.random.default_rng(41)
    st = C.OneBitState.zeros((3000,))
    for k in range(12):
        g = (r.normal(size=3000) * 10.0 ** r.uniform(-3, 0)).astype(np.float32)
        q = C.onebit_quantize(g, st)
        arrays[f"onebit/{k}/g"] = g
        arrays[f"onebit/{k}/bits"] = q.codes.copy()
        arrays[f"onebit/{k}/levels"] = np.array([q.pos_level, q.neg_level], np.float64)
        arrays[f"onebit/{k}/residual"] = st.residual.copy()
        arrays[f"onebit/{k}/decoded"] = C.onebit_decode(q)

    # error suite at the paper's protocol size used by test_acceptance.py:132-149
    reps = EB.run_error_suite(seed=0, count=1_000_000)
    meta["suite"] = [
        {"dist": r.sample_label, "spec": r.spec.label(), "seed": r.seed,
         "mean_abs_error": r.mean_abs_error, "mean_rel_error_pct": r.mean_rel_error_pct}
        for r in reps
    ]

    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
    print("wrote", OUT / "golden.npz", (OUT / "golden.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
