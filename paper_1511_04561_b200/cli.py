"""Command-line front-end of the hot path: the codec subcommands of the
reference CLI (approx8/cli.py:72-128, parser :224-253), same flags, same
A8T1 files (tensorfile.py), same exit codes (cli.py:301-314: 0 success,
1 input/usage problem, 2 configuration problem) -- running on the B200
kernels.

    python -m paper_1511_04561_b200 codebook --dtype dynamic-tree [--norm none] [--out F]
    python -m paper_1511_04561_b200 encode --in F --out G --dtype D [--norm N]
    python -m paper_1511_04561_b200 decode --in G --out H [--dtype D --norm N]
    python -m paper_1511_04561_b200 bench-error [--n N] [--seed S] [--table] [--out F]

The reference's perf-model / trainer subcommands (predict, sweep, train,
parity) are outside this path.
"""

from __future__ import annotations

import argparse
import io
import sys
from pathlib import Path
from typing import Optional

import numpy as np

from . import codecs, tensorfile
from .codecs import DataTypeKind, DataTypeSpec, NormKind
from .errors import ApproxError, ConfigError, InputError, UsageError
from .exchange import ONEBIT

DTYPE_CHOICES = [k.value for k in DataTypeKind] + [ONEBIT]


class _Parser(argparse.ArgumentParser):
    # cli.py:25-29: argparse errors are usage problems (exit 1), not exit 2
    def error(self, message: str):
        raise UsageError(f"{message}\n{self.format_usage().rstrip()}")


def _parse_norm(text: str) -> tuple:
    """cli.py:32-42: none | absmax | decade:N."""
    if text == "none":
        return NormKind.NONE, 0
    if text == "absmax":
        return NormKind.ABSMAX, 0
    if text.startswith("decade:"):
        try:
            return NormKind.DECADE, int(text.split(":", 1)[1])
        except ValueError as exc:
            raise UsageError(f"bad decade offset in --norm {text!r}") from exc
    raise UsageError(f"--norm must be none, absmax, or decade:N, got {text!r}")


def _spec_from_flags(dtype: str, norm: str) -> DataTypeSpec:
    kind = DataTypeKind(dtype)
    norm_kind, decades = _parse_norm(norm)
    return DataTypeSpec(kind, norm_kind, decades)


def _emit(text: str, out: Optional[str]) -> None:
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


def _cmd_codebook(args) -> int:
    if args.dtype == ONEBIT:
        raise UsageError("onebit has no static codebook to dump")
    buf = io.StringIO()
    codecs.build_codebook(_spec_from_flags(args.dtype, args.norm)).dump(buf)
    _emit(buf.getvalue(), args.out)
    return 0


def _cmd_encode(args) -> int:
    """cli.py:87-99: raw float32 file -> 8-bit (or 1-bit) A8T1 file."""
    data = tensorfile.read_tensor(args.infile)
    if not isinstance(data, np.ndarray):
        raise InputError(f"{args.infile} already holds encoded data; expected raw floats")
    if args.dtype == ONEBIT:
        q = codecs.onebit_quantize(data, codecs.OneBitState.zeros(data.shape))
    else:
        q = codecs.encode_buffer(data, codecs.build_codebook(_spec_from_flags(args.dtype, args.norm)))
    tensorfile.write_tensor(args.out, q)
    return 0


def _cmd_decode(args) -> int:
    """cli.py:102-117: encoded A8T1 file -> raw float32 file."""
    data = tensorfile.read_tensor(args.infile)
    if isinstance(data, np.ndarray):
        raise InputError(f"{args.infile} holds raw floats; nothing to decode")
    if data.nbits == 1:
        decoded = codecs.onebit_decode(data)
    else:
        if args.dtype is not None:
            expected = _spec_from_flags(args.dtype, args.norm)
            if expected != data.spec:
                raise InputError(f"{args.infile} was encoded as {data.spec.label()}, flags say {expected.label()}")
        decoded = codecs.decode_buffer(data, codecs.build_codebook(data.spec))
    tensorfile.write_tensor(args.out, decoded)
    return 0


def _cmd_bench_error(args) -> int:
    """cli.py:120-127 on the GPU error bench (errorbench.py)."""
    from . import errorbench

    reports = errorbench.run_error_suite(seed=args.seed, count=args.n)
    _emit(errorbench.format_table(reports) if args.table else errorbench.reports_to_csv(reports), args.out)
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = _Parser(prog="python -m paper_1511_04561_b200",
                     description="8-bit approximation codec on B200 (the approx8 codec CLI)")
    sub = parser.add_subparsers(dest="command", required=True, parser_class=_Parser)

    p = sub.add_parser("codebook", help="print all 256 codes of a data type")
    p.add_argument("--dtype", required=True, choices=DTYPE_CHOICES)
    p.add_argument("--norm", default="none")
    p.add_argument("--out")
    p.set_defaults(func=_cmd_codebook)

    p = sub.add_parser("encode", help="encode a float32 tensor file")
    p.add_argument("--in", dest="infile", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--dtype", required=True, choices=DTYPE_CHOICES)
    p.add_argument("--norm", default="none")
    p.set_defaults(func=_cmd_encode)

    p = sub.add_parser("decode", help="decode an encoded tensor file back to float32")
    p.add_argument("--in", dest="infile", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--dtype", choices=DTYPE_CHOICES)
    p.add_argument("--norm", default="none")
    p.set_defaults(func=_cmd_decode)

    p = sub.add_parser("bench-error", help="distribution x codec error grid")
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--table", action="store_true", help="aligned text instead of CSV")
    p.add_argument("--out")
    p.set_defaults(func=_cmd_bench_error)
    return parser


def main(argv: Optional[list] = None) -> int:
    """cli.py:301-314: ConfigError -> 2, other package errors and OSError -> 1."""
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
        return args.func(args)
    except ConfigError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except ApproxError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
