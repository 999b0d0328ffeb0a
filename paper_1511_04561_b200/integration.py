"""The module-level drop-in of INTEGRATION.md section 1, as code.

A maintainer of the reference package ``approx8`` adds two opt-in blocks:
one at the end of ``approx8/errors.py`` (so every ``approx8`` module and
caller catches the classes this package raises) and one at the end of
``approx8/codecs.py`` (so ``approx8.mlp``, ``approx8.tensorfile``,
``approx8.errorbench``, ``approx8.cli`` and user code bind the B200 codec
when they import it).  Both are inert unless ``APPROX8_BACKEND=b200``.

``patch_reference`` applies exactly these blocks to a copy of an installed
``approx8`` package; the drop-in test (tests/test_dropin_reference.py) runs
the reference's own test-suite against such a copy.
"""

from __future__ import annotations

import shutil
from pathlib import Path

# appended to approx8/errors.py (reference errors.py:16-33 defines the same five classes)
ERRORS_PATCH = '''
# --- B200 backend (paper_1511_04561_b200, INTEGRATION.md section 1) ---
import os as _a8_os
if _a8_os.environ.get("APPROX8_BACKEND") == "b200":
    from paper_1511_04561_b200.errors import (  # noqa: F401,E402  (re-export)
        ApproxError, ConfigError, InputError, TrainingError, UsageError,
    )
'''

# appended to approx8/codecs.py (reference codecs.py:68-348)
CODECS_PATCH = '''
# --- B200 backend (paper_1511_04561_b200, INTEGRATION.md section 1) ---
import os as _a8_os
if _a8_os.environ.get("APPROX8_BACKEND") == "b200":
    from paper_1511_04561_b200.codecs import (  # noqa: F401,E402  (re-export)
        SIGN_MASK, Codebook, DataTypeKind, DataTypeSpec, NormKind, OneBitState, QuantizedTensor,
        build_codebook, decode_buffer, encode_buffer, onebit_decode, onebit_quantize, roundtrip,
    )
    from .errors import ConfigError, InputError, UsageError  # noqa: F401,E402  (now the B200 classes)
'''


def patch_reference(src_pkg: Path, dst_parent: Path) -> Path:
    """Copy the ``approx8`` package directory ``src_pkg`` into ``dst_parent``
    and append the two opt-in blocks.  Returns the new package directory."""
    dst = Path(dst_parent) / "approx8"
    shutil.copytree(src_pkg, dst, ignore=shutil.ignore_patterns("__pycache__"))
    for name, patch in (("errors.py", ERRORS_PATCH), ("codecs.py", CODECS_PATCH)):
        with open(dst / name, "a") as f:
            f.write(patch)
    return dst
