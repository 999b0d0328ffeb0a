"""Test-only helpers: golden fixtures, a NumPy ``SegmentCodec`` built on the
oracle (used ONLY to exercise the exchange orchestration on CPU/gloo), and a
thread-based virtual-rank comm for multi-rank tests inside one process."""

from __future__ import annotations

import hashlib
import json
import sys
import threading
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from oracle import approx8_oracle as O  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


_cache: dict = {}


def golden():
    if "g" not in _cache:
        _cache["g"] = (np.load(GOLDEN / "golden.npz"), json.loads((GOLDEN / "golden.json").read_text()))
    return _cache["g"]


def parse_tag(tag: str):
    """'mantissa/decade+2' -> ('mantissa', 'decade', 2)."""
    kind, _, norm = tag.partition("/")
    if norm.startswith("decade"):
        return kind, "decade", int(norm[6:])
    return kind, norm or "none", 0


def golden_cases():
    """(name, spec tuple, x, reference codes) for every stored vector case."""
    g, _ = golden()
    out = []
    for key in sorted(g.files):
        if not key.endswith("/x") or key.startswith("full/"):
            continue
        base = key[:-2]
        parts = base.split("/")
        if parts[0] in ("scan", "adv"):
            spec = parse_tag("/".join(parts[1:3]))
        elif parts[0] == "extreme":
            spec = (parts[1], "absmax", 0)
        else:
            continue
        out.append((base, spec, g[key], g[base + "/codes"]))
    return out


def fullrange_cases():
    """Buffers of 1..24 finite float32 patterns per spec (hypothesis domain)."""
    g, _ = golden()
    out = []
    for key in sorted(g.files):
        if key.startswith("full/") and key.endswith("/x"):
            base = key[:-2]
            spec = parse_tag(base[5:])
            sizes = g[base + "/sizes"]
            xs = np.split(g[key], np.cumsum(sizes)[:-1])
            cs = np.split(g[base + "/codes"], np.cumsum(sizes)[:-1])
            out.append((base, spec, xs, cs, g[base + "/scales"]))
    return out


def acceptance_inputs():
    """test_acceptance.py:116-129 inputs, regenerated from the same rng stream."""
    rng = np.random.default_rng(20240818)
    specs = [("dynamic-tree", "absmax", 0), ("static-tree", "none", 0),
             ("mantissa", "none", 0), ("linear", "absmax", 0)]
    out = []
    for spec in specs:
        mags = 10.0 ** rng.uniform(-8.0, 3.0, size=100_000)
        x = (mags * rng.choice([-1.0, 1.0], size=mags.size)).astype(np.float32)
        out.append((spec, x))
    return out


def tag(spec) -> str:
    kind, norm, dec = spec
    return f"{kind}/{norm}{dec:+d}" if norm == "decade" else f"{kind}/{norm}"


# ---------------------------------------------------------------------------
# NumPy codec backend (test-only; mirrors the byte layout of the C ABI)


class NumpyCodec:
    """Implements exchange.SegmentCodec with the oracle on CPU tensors."""

    def __init__(self, spec):
        self.kind = spec.kind.value
        self.norm = spec.normalization.value
        self.dec = spec.decades

    @staticmethod
    def _addr(codes_off, e, L, stride):
        return codes_off + (e // L) * stride + (e % L)

    def encode(self, xs, flat_offs, scale_idx, cb, buf, codes_off, scales_off, block_len,
               block_stride, scale_block_stride, reps, status_off, status_in=None):
        mem = buf.numpy()
        status = 0
        for x, f0, si in zip(xs, flat_offs, scale_idx):
            xn = x.detach().cpu().numpy().ravel()
            try:
                codes, s = O.encode(xn, self.kind, self.norm, self.dec)
            except O.NonFinite:
                status |= 1
                codes = np.zeros(xn.size, np.uint8)
                s = O.scale_of(xn[np.isfinite(xn)], self.norm, self.dec)
            e = np.arange(xn.size, dtype=np.int64) + f0
            mem[self._addr(codes_off, e, block_len, block_stride)] = codes
            for k in range(reps):
                at = scales_off + 4 * (k * scale_block_stride + si)
                mem[at:at + 4] = np.frombuffer(np.float32(s).tobytes(), np.uint8)
        if status_in is not None:
            status |= int(status_in.view(torch.int32)[0])
        for k in range(reps):
            at = status_off + 4 * k * scale_block_stride
            mem[at:at + 4] = np.frombuffer(np.uint32(status).tobytes(), np.uint8)

    def decode(self, outs, flat_offs, scale_idx, cb, buf, codes_off, scales_off, block_len,
               block_stride, scale_block_stride, rank_stride, nranks, op, status_idx=-1,
               status_blocks=0, status_out=None, locals_=None, local_rank=-1, status_count=False):
        mem = buf.numpy()
        table = O.book(self.kind).table
        for i, (o, f0, si) in enumerate(zip(outs, flat_offs, scale_idx)):
            n = o.numel()
            if n == 0:
                continue
            e = np.arange(n, dtype=np.int64) + f0
            j = f0 // block_len
            acc = None
            for r in range(nranks):
                c = mem[r * rank_stride + self._addr(codes_off, e, block_len, block_stride)]
                at = r * rank_stride + scales_off + 4 * (j * scale_block_stride + si)
                s = np.frombuffer(mem[at:at + 4].tobytes(), np.float32)[0]
                d = table[c] * np.float32(s)
                if locals_ is not None and r == local_rank:
                    d = locals_[i].reshape(-1).numpy().astype(np.float32)
                acc = d.copy() if acc is None else (acc + d).astype(np.float32)
            if op == 1:
                acc = (acc / np.float32(nranks)).astype(np.float32)
            o.view(-1).copy_(torch.from_numpy(acc))
        if status_out is not None:
            st = 0
            for r in range(nranks):
                for j in range(status_blocks):
                    at = r * rank_stride + scales_off + 4 * (j * scale_block_stride + status_idx)
                    st |= int(np.frombuffer(mem[at:at + 4].tobytes(), np.uint32)[0])
            w = status_out.view(torch.int32)
            if status_count:
                w[0] = int(w[0]) + (1 if st else 0)
            else:
                w[0] = st


class NumpyOneBitCodec:
    """The 1-bit half of exchange.SegmentCodec (onebit_quantize /
    onebit_reduce) with the oracle on CPU tensors, same slab byte layout."""

    def onebit_quantize(self, x, residual, buf, bits_off, levels_off, status_off):
        mem = buf.numpy()
        xn = x.detach().cpu().numpy().ravel()
        res = residual.numpy()
        try:
            bits, pos, neg, new = O.onebit_quantize(xn, res)
            residual.copy_(torch.from_numpy(new))
            st = 0
        except O.NonFinite:
            bits, pos, neg, st = np.zeros((xn.size + 7) // 8, np.uint8), 0.0, 0.0, 1
        mem[bits_off:bits_off + bits.size] = bits
        mem[levels_off:levels_off + 8] = np.frombuffer(np.array([pos, neg], np.float32).tobytes(), np.uint8)
        mem[status_off:status_off + 4] = np.frombuffer(np.uint32(st).tobytes(), np.uint8)

    def onebit_reduce(self, outs, bit_offs, buf, rank_stride, levels_off, status_off, nranks, op, status_out=None):
        mem = buf.numpy()
        for i, (o, bo) in enumerate(zip(outs, bit_offs)):
            n = o.numel()
            acc = None
            for r in range(nranks):
                base = r * rank_stride
                lv = np.frombuffer(mem[base + levels_off + 8 * i:base + levels_off + 8 * i + 8].tobytes(), np.float32)
                d = O.onebit_decode(mem[base + bo:base + bo + (n + 7) // 8], n, float(lv[0]), float(lv[1]))
                acc = d.astype(np.float32) if acc is None else (acc + d).astype(np.float32)
            if op == 1 and acc is not None:
                acc = (acc / np.float32(nranks)).astype(np.float32)
            if n:
                o.view(-1).copy_(torch.from_numpy(acc))
        if status_out is not None:
            st = 0
            for r in range(nranks):
                for i in range(len(outs)):
                    at = r * rank_stride + status_off + 4 * i
                    st |= int(np.frombuffer(mem[at:at + 4].tobytes(), np.uint32)[0])
            status_out.view(torch.int32)[0] = st


# ---------------------------------------------------------------------------
# virtual ranks: one thread per rank, collectives through shared memory


class ThreadComm:
    """all_gather / all_to_all between threads of one process.  Synchronises
    the CUDA device around every exchange of buffers."""

    class _Shared:
        def __init__(self, n):
            self.n = n
            self.barrier = threading.Barrier(n)
            self.slots = [None] * n

    def __init__(self, shared, rank):
        self.s = shared
        self.rank = rank

    @classmethod
    def group(cls, n):
        sh = cls._Shared(n)
        return [cls(sh, r) for r in range(n)]

    def world(self):
        return self.s.n, self.rank

    def _sync(self, t):
        if t.is_cuda:
            torch.cuda.synchronize(t.device)

    def all_gather(self, out, slot):
        self._sync(slot)
        self.s.slots[self.rank] = slot.clone()
        self.s.barrier.wait()
        out.copy_(torch.cat([x.to(out.device) for x in self.s.slots]))
        self._sync(out)
        self.s.barrier.wait()

    def all_to_all(self, recv, send):
        self._sync(send)
        self.s.slots[self.rank] = send.clone()
        self.s.barrier.wait()
        n = self.s.n
        blk = send.numel() // n
        parts = [self.s.slots[r][self.rank * blk:(self.rank + 1) * blk].to(recv.device) for r in range(n)]
        recv.copy_(torch.cat(parts))
        self._sync(recv)
        self.s.barrier.wait()


class VirtualPeers:
    """exchange.PeerTransport between threads on ONE GPU: every virtual
    rank's buffer is an ordinary allocation whose address the others read
    directly (what NVLink peer mappings give real ranks)."""

    class _Shared:
        def __init__(self, n):
            self.n = n
            self.barrier = threading.Barrier(n)
            self.bufs = {}
            self.lock = threading.Lock()

    def __init__(self, shared, rank):
        self.s = shared
        self.rank = rank
        self._mine = {}

    @classmethod
    def group(cls, n):
        sh = cls._Shared(n)
        return [cls(sh, r) for r in range(n)]

    def world(self):
        return self.s.n, self.rank

    def buffer(self, name, nbytes, device):
        hit = self._mine.get(name)
        if hit is None or hit[0].numel() < nbytes:
            t = torch.zeros(max(int(nbytes), 16), dtype=torch.uint8, device=device)
            with self.s.lock:
                self.s.bufs.setdefault(name, [None] * self.s.n)[self.rank] = t
            self.s.barrier.wait()
            ptrs = [b.data_ptr() for b in self.s.bufs[name]]
            self.s.barrier.wait()
            hit = self._mine[name] = (t, ptrs)
        return hit[0][:nbytes], hit[1]

    def barrier(self):
        torch.cuda.synchronize()
        self.s.barrier.wait()


def run_virtual_peers(n, fn):
    """Run fn(rank, peers) in n threads with VirtualPeers transports."""
    peers = VirtualPeers.group(n)
    res = [None] * n
    errs = []

    def body(r):
        try:
            res[r] = fn(r, peers[r])
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            peers[r].s.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res


def run_virtual_ranks(n, fn):
    """Run fn(rank, comm) in n threads; return the per-rank results."""
    comms = ThreadComm.group(n)
    res = [None] * n
    errs = []

    def body(r):
        try:
            res[r] = fn(r, comms[r])
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            comms[r].s.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res
