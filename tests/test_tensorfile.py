"""A8T1 tensor files: byte-identical with the reference's writer and
readable from reference-written files (approx8/tensorfile.py).  The golden
files were written by the real reference (tests/golden/make_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from helpers import O, golden, sha

import paper_1511_04561_b200 as A
from paper_1511_04561_b200 import tensorfile as TF

SPECS = [("dynamic-tree", "absmax", 0), ("mantissa", "decade", -2), ("linear", "none", 0)]


def tag(spec):
    kind, norm, dec = spec
    return f"{kind}/{norm}{dec:+d}" if norm == "decade" else f"{kind}/{norm}"


def test_float32_file_is_byte_identical(tmp_path):
    g, _ = golden()
    x = g["a8t1/small_x"]
    assert TF.encode_file_bytes(x) == g["a8t1/float32"].tobytes()
    TF.write_tensor(tmp_path / "f.a8t", torch.from_numpy(x))
    assert (tmp_path / "f.a8t").read_bytes() == g["a8t1/float32"].tobytes()
    back = TF.read_tensor(tmp_path / "f.a8t")
    assert back.dtype == np.float32 and np.array_equal(back, x)


@pytest.mark.parametrize("spec", SPECS, ids=tag)
def test_code_files_match_reference(spec, tmp_path):
    g, _ = golden()
    x = g["a8t1/small_x"]
    codes, s = O.encode(x, *spec)
    q = A.QuantizedTensor(codes, x.shape, A.DataTypeSpec(*spec), s)
    ref = g[f"a8t1/codes/{tag(spec)}"].tobytes()
    assert TF.encode_file_bytes(q) == ref
    (tmp_path / "q.a8t").write_bytes(ref)
    r = TF.read_tensor(tmp_path / "q.a8t")
    assert r.shape == x.shape and r.spec == A.DataTypeSpec(*spec) and r.scale == s
    assert np.array_equal(r.codes_numpy(), codes)


def test_onebit_file_roundtrip():
    g, _ = golden()
    ref = g["a8t1/onebit"].tobytes()
    q = TF.decode_file_bytes(ref)
    assert q.nbits == 1 and q.spec is None and q.shape == (3, 4, 5)
    assert TF.encode_file_bytes(q) == ref


def test_malformed_files_raise_input_error():
    g, _ = golden()
    good = g["a8t1/float32"].tobytes()
    bad = [b"XXXX" + good[4:], good[:6], good[:-1], good[:4] + bytes([7]) + good[5:],
           good[:5] + bytes([9]) + good[6:], good[:6] + bytes([5]) + good[7:], good[:8] + bytes([9]) + good[9:]]
    for b in bad:
        with pytest.raises(A.InputError):
            TF.decode_file_bytes(b)
    q = A.QuantizedTensor(np.zeros(1, np.uint8), (1,) * 9, A.DataTypeSpec("linear"), 1.0)
    with pytest.raises(A.UsageError):
        TF.encode_file_bytes(q)


@pytest.mark.gpu
def test_gpu_codes_written_as_reference_files(cuda):
    g, meta = golden()
    x = g["a8t1/small_x"]
    for spec in SPECS:
        q = A.encode_buffer(torch.from_numpy(x).to(cuda), A.build_codebook(A.DataTypeSpec(*spec)))
        assert TF.encode_file_bytes(q) == g[f"a8t1/codes/{tag(spec)}"].tobytes(), spec
    x1 = O.sample_normal(2**20, 0)
    q = A.encode_buffer(torch.from_numpy(x1).to(cuda), A.build_codebook(A.DataTypeSpec("dynamic-tree", "absmax")))
    assert sha(np.frombuffer(TF.encode_file_bytes(q), np.uint8)) == meta["a8t1"]["c1_dynamic_absmax_sha"]
    # and a reference file decodes on the GPU to the reference values
    r = TF.decode_file_bytes(g["a8t1/codes/dynamic-tree/absmax"].tobytes())
    y = A.decode_buffer(r, A.build_codebook(r.spec), device=cuda)
    assert isinstance(y, np.ndarray)  # host codes decode to NumPy, as in the reference
    assert y.tobytes() == O.roundtrip(x, "dynamic-tree", "absmax").tobytes()
