"""The codec CLI mirror (paper_1511_04561_b200/cli.py) against the
reference CLI's behaviour (approx8/cli.py:72-128, exit codes :301-314; the
reference's own tests pkg/tests/test_cli.py:40-170 are the model).  Files
are A8T1 (tensorfile.py) and byte-identical to the reference's."""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from helpers import O, golden, tag

import paper_1511_04561_b200 as A
from paper_1511_04561_b200 import tensorfile as TF
from paper_1511_04561_b200.cli import main

ROOT = Path(__file__).resolve().parents[1]


def test_unknown_flag_and_subcommand_are_usage_errors(capsys):
    assert main(["codebook", "--dtype", "linear", "--bogus"]) == 1
    assert main(["frobnicate"]) == 1
    assert main(["encode", "--in", "x"]) == 1  # missing required flags
    assert "error" in capsys.readouterr().err


def test_domain_violation_is_config_error(capsys):
    assert main(["codebook", "--dtype", "static-tree", "--norm", "absmax"]) == 2
    assert "configuration error" in capsys.readouterr().err


def test_bad_decade_offset_is_usage_error():
    assert main(["codebook", "--dtype", "mantissa", "--norm", "decade:x"]) == 1


def test_missing_input_file(tmp_path):
    assert main(["encode", "--in", str(tmp_path / "nope.bin"), "--out", str(tmp_path / "o"), "--dtype", "linear"]) == 1


def test_codebook_dump_matches_reference_format(capsys):
    assert main(["codebook", "--dtype", "dynamic-tree"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert len(lines) == 256 and lines[1] == "0x01\t5.49999982e-07"  # %.9g of float32(5.5e-7), codecs.py:180-183
    assert main(["codebook", "--dtype", "onebit"]) == 1


def test_decode_raw_input_rejected(tmp_path):
    src = tmp_path / "s.bin"
    TF.write_tensor(src, np.ones(4, dtype=np.float32))
    assert main(["decode", "--in", str(src), "--out", str(tmp_path / "o.bin")]) == 1


def test_module_entry_point():
    out = subprocess.run([sys.executable, "-m", "paper_1511_04561_b200", "codebook", "--dtype", "linear"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.count("\n") == 256


@pytest.mark.gpu
def test_encode_decode_files_match_reference(tmp_path, cuda):
    """encode writes the reference's A8T1 bytes (goldens from the real
    reference); decode of a reference file gives the reference values."""
    g, meta = golden()
    x = g["a8t1/small_x"]
    src = tmp_path / "x.bin"
    TF.write_tensor(src, x)
    for spec in (("dynamic-tree", "absmax", 0), ("mantissa", "decade", -2), ("linear", "none", 0)):
        norm = f"decade:{spec[2]}" if spec[1] == "decade" else spec[1]
        out = tmp_path / f"{spec[0]}.a8t"
        assert main(["encode", "--in", str(src), "--out", str(out), "--dtype", spec[0], "--norm", norm]) == 0
        assert out.read_bytes() == g[f"a8t1/codes/{tag(spec)}"].tobytes(), spec
        back = tmp_path / f"{spec[0]}.f32"
        assert main(["decode", "--in", str(out), "--out", str(back)]) == 0
        want = O.roundtrip(x, spec[0], spec[1], spec[2]).astype(np.float32)
        assert TF.read_tensor(back).tobytes() == want.tobytes(), spec
    # flag mismatch on decode: InputError -> exit 1
    coded = tmp_path / "dynamic-tree.a8t"
    assert main(["decode", "--in", str(coded), "--out", str(tmp_path / "z"), "--dtype", "mantissa"]) == 1
    # encoded input to encode: exit 1
    assert main(["encode", "--in", str(coded), "--out", str(tmp_path / "z"), "--dtype", "linear"]) == 1


@pytest.mark.gpu
def test_onebit_cli_roundtrip(tmp_path, cuda):
    g = np.random.default_rng(3).normal(size=(6, 4)).astype(np.float32)
    src, coded, back = (tmp_path / n for n in ("s.bin", "c.bin", "b.bin"))
    TF.write_tensor(src, g)
    assert main(["encode", "--in", str(src), "--out", str(coded), "--dtype", "onebit"]) == 0
    assert main(["decode", "--in", str(coded), "--out", str(back)]) == 0
    bits, pos, neg, _ = O.onebit_quantize(g, np.zeros(g.shape))
    want = O.onebit_decode(bits, g.size, pos, neg).reshape(g.shape)
    assert TF.read_tensor(back).tobytes() == want.tobytes()
