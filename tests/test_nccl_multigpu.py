"""The N > 1 exchange on real NCCL (one process per GPU): tools/nccl_parity.py
under torchrun, at 2 GPUs and at every visible GPU.  Skipped below 2 GPUs
(the round-end GPU tier has one; the scaling box has 8)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("nproc", [2, 0])
def test_nccl_exchange_parity(nproc):
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    n = nproc or ngpu
    if nproc == 0 and ngpu == 2:
        pytest.skip("covered by nproc=2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tools" / "nccl_parity.py")]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500,
                         env=dict(os.environ, A8_PARITY_C3="1"))
    lines = [json.loads(ln) for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert res.returncode == 0 and len(lines) == n, res.stdout[-3000:] + res.stderr[-3000:]
    for ln in lines:
        assert ln["ok"] and ln["backend"] == "nccl", ln
