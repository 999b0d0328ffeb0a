"""Build the sm_100a C-ABI library in-tree with nvcc (no JIT, no torch build).

    python paper_1511_04561_b200/build.py [--force] [-v]   # -> paper_1511_04561_b200/_lib/libapprox8_b200.so

(Run it as a script: importing the package loads the library it builds.)

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libapprox8_b200.so"
INCLUDE = ROOT / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES = ["a8_kernels.cu", "a8_onebit.cu", "a8_errstats.cu", "a8_blocked.cu", "a8_produce.cu", "a8_codebook.cpp"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the approx8 B200 library needs the CUDA toolkit to build")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, ticket_trace: bool = False, defines=(), variant: str = "") -> Path:
    """``ticket_trace``: a debug build with per-ticket timestamps into
    ``_lib_trace/`` (load it with A8_LIB=<path>); never the product library.
    ``defines`` + ``variant``: a tuning build (-D flags) into ``_lib_var/<variant>/``
    for A/B measurements; never the product library."""
    if variant:
        lib = PKG / "_lib_var" / variant / LIB.name
    else:
        lib = (PKG / "_lib_trace" / LIB.name) if ticket_trace else LIB
    if not force and not ticket_trace and not variant and not _stale():
        return LIB
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    cmd = [
        nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo",
        "-Xcompiler", "-fPIC,-O3", "-shared", "-cudart", "static",
        "-Xptxas", "-v" if verbose else "-O3",
        f"-I{INCLUDE}", f"-I{CSRC}", *(["-DA8_TICKET_TRACE"] if ticket_trace else []), *[f"-D{d}" for d in defines],
        *[str(CSRC / s) for s in SOURCES],
        "-o", str(tmp),
    ]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stdout + res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    var = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, ticket_trace="--ticket-trace" in sys.argv,
                defines=defs, variant=var))
