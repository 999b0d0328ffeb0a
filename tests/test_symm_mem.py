"""PeerExchange on torch.distributed._symmetric_memory (NVLink peer
mappings), one process (the transport, rendezvous, device barrier and
a8_decode_peers path end to end at world size 1; tools/nccl_parity.py covers
N > 1 on a multi-GPU box)."""

from __future__ import annotations

import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu

SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {root!r})
import paper_1511_04561_b200 as A
from oracle import approx8_oracle as O
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="{port}")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
ex = A.PeerExchange(A.DataTypeSpec("dynamic-tree", "absmax"), A.SymmetricMemoryTransport(), check="sync")
rng = np.random.default_rng(0)
for step in range(3):
    gs = [rng.normal(0, 1e-2, n).astype(np.float32) for n in (1000, 17, 70000, 5)]
    ts = [torch.from_numpy(g).to(dev) for g in gs]
    ex(ts)
    for t, g in zip(ts, gs):
        assert t.cpu().numpy().tobytes() == O.roundtrip(g, "dynamic-tree", "absmax").tobytes(), step
dist.destroy_process_group()
print("symm ok")
"""


def test_symmetric_memory_peer_exchange_world_1():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), port=port)], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "symm ok" in res.stdout, res.stdout[-2000:] + res.stderr[-3000:]
