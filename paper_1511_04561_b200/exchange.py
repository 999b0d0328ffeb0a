"""Compressed gradient exchange (data parallel) over NCCL, 8-bit on the wire.

The reference has no multi-process exchange: its data-parallel seam rounds
every W and b gradient through encode->decode just before the optimizer step
(approx8/mlp.py:167-175, 322-325, 367-369), i.e. it simulates "each GPU
receives the 8-bit gradients of the others".  This module is that exchange
for real, one process per GPU:

``allgather`` (north star item 4)
    every rank encodes each tensor with its own per-tensor scale into one
    slab [codes of all tensors | scales | status], the slabs are all-gathered
    in place with NCCL over NVLink, and one fused kernel decodes the N slabs,
    sums them in rank order in float32 and divides by N.
    Per-rank ingress (N-1)*n bytes (vs 2(N-1)/N*4n for a ring fp32 all-reduce).

``two_round`` (the paper's scatter + broadcast, PAPER.md:380,
perfmodel.py:246-273)
    round 1 all-to-all of 8-bit shards, fused decode-average of the N
    contributions to the local shard, re-encode of the shard with one scale
    per (tensor x shard) piece, round 2 all-gather of the 8-bit shards, decode.
    Per-rank ingress 2(N-1)/N*n bytes.

Exchange semantics (the composed oracles in oracle/approx8_oracle.py):
  * allgather: out = fl32(sum_r decode(encode(g_r))) / N, rank order;
  * two_round: out = decode(encode(piece of allgather-average)) per piece;
  * world size 1: out == roundtrip(g) bit for bit.

The codec work goes through a ``SegmentCodec``; the default is the CUDA
library.  The orchestration (layouts, collectives, status propagation) is
independent of it, which is what the CPU gloo tests exercise.
"""

from __future__ import annotations

import collections
import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch
import torch.distributed as dist

from . import _native as N
from .codecs import Codebook, DataTypeSpec, build_codebook, round16, workspace, workspace_epoch
from .errors import InputError, UsageError

MODES = ("allgather", "two_round")
OPS = ("avg", "sum")
ONEBIT = "onebit"  # the 1-bit error-feedback spec of the DP seam (mlp.py:52, 313-321)


# ---------------------------------------------------------------------------
# codec backends


class SegmentCodec:
    """Interface of the codec work the exchange needs.  Buffers are uint8
    tensors; offsets are bytes; strides follow include/approx8_b200.h."""

    def encode(self, xs, flat_offs, scale_idx, cb: Codebook, buf: torch.Tensor, codes_off: int,
               scales_off: int, block_len: int, block_stride: int, scale_block_stride: int,
               reps: int, status_off: int, status_in: Optional[torch.Tensor] = None,
               amax: Optional[torch.Tensor] = None) -> None:
        """``amax``: float32 device tensor, max|xs[i]| per tensor as written by
        the producer (absmax specs): one-pass encode (a8_encode_premax)."""
        raise NotImplementedError

    def decode(self, outs, flat_offs, scale_idx, cb: Codebook, buf: torch.Tensor, codes_off: int,
               scales_off: int, block_len: int, block_stride: int, scale_block_stride: int,
               rank_stride: int, nranks: int, op: int, status_idx: int = -1,
               status_blocks: int = 0, status_out: Optional[torch.Tensor] = None,
               locals_: Optional[Sequence[torch.Tensor]] = None, local_rank: int = -1,
               status_count: bool = False) -> None:
        """``locals_``: rank ``local_rank``'s term of output i is locals_[i]
        (float32, outs[i].numel() elements) instead of its decoded codes.
        ``status_count``: increment ``status_out`` when the status is non-zero
        instead of overwriting it (A8_LAYOUT_STATUS_COUNT)."""
        raise NotImplementedError


class CudaSegmentCodec(SegmentCodec):
    """a8_encode / a8_decode (and the 1-bit a8_onebit_quantize /
    a8_onebit_reduce) on the buffers' device and current stream."""

    _lib = N.lib  # a recording proxy while GradientExchange prepares a step (see _StepRecorder)

    def decode_peers(self, outs, flat_offs, scale_idx, cb, codes_rel, scales_rel, block_len, block_stride,
                     scale_block_stride, rank_bases, op, status_idx=-1, status_blocks=0, status_out=None):
        """a8_decode_peers: rank r's codes at rank_bases[r] + codes_rel and its
        scales at rank_bases[r] + scales_rel (device addresses, e.g. NVLink
        peer mappings); the sum over ranks in rank order, then op."""
        dev = outs[0].device if outs else status_out.device
        book, _ = cb.device_tables(dev)
        n = len(outs)
        segs = (N.DecSeg * max(n, 1))()
        for i, (o, off, si) in enumerate(zip(outs, flat_offs, scale_idx)):
            segs[i] = N.DecSeg(o.data_ptr(), o.numel(), off, si, 0)
        b0 = int(rank_bases[0])
        lay = N.Layout(b0 + codes_rel, b0 + scales_rel, block_len, block_stride, scale_block_stride, 0, 1, 0)
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = workspace(dev, stream, max(n, 1))
        bases = (C.c_void_p * len(rank_bases))(*[int(b) for b in rank_bases])
        st = None if status_out is None else status_out.data_ptr()
        N.check(N.lib.a8_decode_peers(segs, n, book.data_ptr(), lay, bases, len(rank_bases), op, status_idx,
                                      status_blocks, st, ws.data_ptr(), ws.numel(), stream))

    def onebit_quantize(self, x: torch.Tensor, residual: torch.Tensor, buf: torch.Tensor, bits_off: int,
                        levels_off: int, status_off: int) -> None:
        """onebit_quantize (codecs.py:306-339) of x with the float64 device
        residual (updated in place), bits / levels / status into buf."""
        from .codecs import _ob_ws

        dev = buf.device
        n = x.numel()
        base = buf.data_ptr()
        stream = torch.cuda.current_stream(dev).cuda_stream
        if n == 0:
            buf[levels_off:levels_off + 12].zero_()
            return
        ws = _ob_ws.get(dev.index)
        if ws is None:
            ws = _ob_ws[dev.index] = torch.empty(N.lib.a8_onebit_workspace_bytes(), dtype=torch.uint8, device=dev)
        N.check(N.lib.a8_onebit_quantize(x.data_ptr(), 1 if x.dtype == torch.float64 else 0, residual.data_ptr(), n,
                                         base + bits_off, base + levels_off, base + status_off, ws.data_ptr(),
                                         ws.numel(), stream))

    def onebit_quantize_many(self, xs, residuals, buf: torch.Tensor, bits_offs, levels_offs, status_offs) -> None:
        """onebit_quantize of every tensor in two launches per 32 tensors of
        one dtype (a8_onebit_quantize_multi; bit-identical per tensor)."""
        dev = buf.device
        base = buf.data_ptr()
        stream = torch.cuda.current_stream(dev).cuda_stream
        groups: dict = {}
        for i, x in enumerate(xs):
            groups.setdefault(x.dtype == torch.float64, []).append(i)
        for f64, idx in groups.items():
            for c0 in range(0, len(idx), 32):
                chunk = idx[c0:c0 + 32]
                segs = (N.ObQSeg * len(chunk))()
                for k, i in enumerate(chunk):
                    x = xs[i]
                    segs[k] = N.ObQSeg(x.data_ptr() if x.numel() else 0, residuals[i].data_ptr() if x.numel() else 0,
                                       x.numel(), base + bits_offs[i], base + levels_offs[i], base + status_offs[i])
                ws = _ob_multi_ws(dev, len(chunk))
                N.check(self._lib.a8_onebit_quantize_multi(segs, len(chunk), 1 if f64 else 0, ws.data_ptr(),
                                                           ws.numel(), stream))

    def onebit_reduce(self, outs, bit_offs, buf: torch.Tensor, rank_stride: int, levels_off: int, status_off: int,
                      nranks: int, op: int, status_out: Optional[torch.Tensor] = None) -> None:
        dev = buf.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        for c0 in range(0, max(len(outs), 1), 32):  # <= 32 segments per launch
            chunk = list(range(c0, min(c0 + 32, len(outs))))
            segs = (N.ObSeg * max(len(chunk), 1))()
            for k, i in enumerate(chunk):
                segs[k] = N.ObSeg(outs[i].data_ptr(), outs[i].numel(), bit_offs[i])
            last = c0 + 32 >= len(outs)
            # the status words of every segment are ORed by the last launch
            N.check(N.lib.a8_onebit_reduce(segs, len(chunk), buf.data_ptr(), rank_stride, levels_off + 8 * c0,
                                           status_off, len(outs) if last else 0, nranks, op,
                                           None if (status_out is None or not last) else status_out.data_ptr(),
                                           stream))

    def encode(self, xs, flat_offs, scale_idx, cb, buf, codes_off, scales_off, block_len,
               block_stride, scale_block_stride, reps, status_off, status_in=None, amax=None):
        dev = buf.device
        book, lut = cb.device_tables(dev)
        n = len(xs)
        segs = (N.EncSeg * n)()
        for i, (x, off, si) in enumerate(zip(xs, flat_offs, scale_idx)):
            segs[i] = N.EncSeg(x.data_ptr(), x.numel(), off, si, 0)
        base = buf.data_ptr()
        lay = N.Layout(base + codes_off, base + scales_off, block_len, block_stride,
                       scale_block_stride, 0, reps, 0)
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = workspace(dev, stream, n)
        if amax is not None:
            N.check(self._lib.a8_encode_premax(segs, n, book.data_ptr(), amax.data_ptr(), lay, ws.data_ptr(),
                                               ws.numel(), None if status_in is None else status_in.data_ptr(),
                                               base + status_off, stream))
            return
        N.check(self._lib.a8_encode(segs, n, book.data_ptr(), cb.spec.norm_code,
                                None if lut is None else lut.data_ptr(), lay, ws.data_ptr(), ws.numel(),
                                None if status_in is None else status_in.data_ptr(),
                                base + status_off, stream))

    def decode(self, outs, flat_offs, scale_idx, cb, buf, codes_off, scales_off, block_len,
               block_stride, scale_block_stride, rank_stride, nranks, op, status_idx=-1,
               status_blocks=0, status_out=None, locals_=None, local_rank=-1, status_count=False):
        dev = buf.device
        book, _ = cb.device_tables(dev)
        n = len(outs)
        segs = (N.DecSeg * max(n, 1))()
        for i, (o, off, si) in enumerate(zip(outs, flat_offs, scale_idx)):
            segs[i] = N.DecSeg(o.data_ptr(), o.numel(), off, si, 0)
        base = buf.data_ptr()
        lay = N.Layout(base + codes_off, base + scales_off, block_len, block_stride,
                       scale_block_stride, rank_stride, 1, N.A8_LAYOUT_STATUS_COUNT if status_count else 0)
        stream = torch.cuda.current_stream(dev).cuda_stream
        ws = workspace(dev, stream, max(n, 1))
        st = None if status_out is None else status_out.data_ptr()
        if locals_ is None:
            N.check(self._lib.a8_decode(segs, n, book.data_ptr(), lay, nranks, op, status_idx,
                                    status_blocks, st, ws.data_ptr(), ws.numel(), stream))
            return
        lp = (C.c_void_p * max(n, 1))(*[t.data_ptr() for t in locals_])
        N.check(self._lib.a8_decode_local(segs, lp, local_rank, n, book.data_ptr(), lay, nranks, op, status_idx,
                                      status_blocks, st, ws.data_ptr(), ws.numel(), stream))


# ---------------------------------------------------------------------------
# collectives


_ob_multi: dict = {}  # device index -> workspace of a8_onebit_quantize_multi (32 segments)


def _ob_multi_ws(dev, nseg: int) -> torch.Tensor:
    ws = _ob_multi.get(dev.index)
    if ws is None:
        ws = _ob_multi[dev.index] = torch.empty(N.lib.a8_onebit_multi_workspace_bytes(32), dtype=torch.uint8,
                                                device=dev)
    return ws


class TorchDistComm:
    """Collectives through ``torch.distributed`` (NCCL over NVLink on the GPU
    box, gloo in the CPU tests).  NCCL runs the all-gather in place."""

    def __init__(self, group=None):
        self.group = group

    def world(self):
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group), dist.get_rank(self.group)
        return 1, 0

    def _inplace(self) -> bool:
        return dist.get_backend(self.group) == "nccl"

    def all_gather(self, out: torch.Tensor, slot: torch.Tensor) -> None:
        dist.all_gather_into_tensor(out, slot if self._inplace() else slot.clone(), group=self.group)

    def all_gather_async(self, out: torch.Tensor, slot: torch.Tensor):
        """Start the all-gather; ``.wait()`` on the result makes the current
        stream wait for it (NCCL: no host block)."""
        return dist.all_gather_into_tensor(out, slot if self._inplace() else slot.clone(), group=self.group,
                                           async_op=True)

    def all_to_all(self, recv: torch.Tensor, send: torch.Tensor) -> None:
        dist.all_to_all_single(recv, send, group=self.group)


# ---------------------------------------------------------------------------
# layouts


@dataclass
class Piece:
    tensor: int  # index of the tensor
    start: int  # first element inside the tensor
    n: int
    flat: int  # global flat index of the first element
    shard: int
    idx: int  # scale slot inside its shard's block


@dataclass
class Plan:
    sizes: tuple
    nranks: int
    offs: list  # flat offset of each tensor (multiples of 16)
    flat: int  # padded flat length (allgather: one block)
    shard: int  # two_round: elements per shard (multiple of 16)
    gap: int  # bytes of scale+status area per block
    nseg: int
    pieces: list = field(default_factory=list)  # two_round pieces, by shard

    @property
    def status_slot(self) -> int:  # index (in 4-byte words) of the status word in a scale area
        return self.nseg

    def allgather_block(self) -> int:
        return self.flat + self.gap

    def two_round_block(self) -> int:
        return self.shard + self.gap


def make_plan(sizes: Sequence[int], nranks: int) -> Plan:
    offs, pos = [], 0
    for n in sizes:
        offs.append(pos)
        pos += round16(n)
    flat = max(pos, 16)
    unit = 16 * nranks
    shard = -(-flat // unit) * unit // nranks
    npieces_max = len(sizes) + nranks
    gap = round16(4 * (max(len(sizes), npieces_max) + 1))
    plan = Plan(tuple(sizes), nranks, offs, round16(flat), shard, gap, len(sizes))
    # two_round pieces: tensor ∩ shard
    per_shard = [0] * nranks
    for t, n in enumerate(sizes):
        a = 0
        while a < n:
            f = offs[t] + a
            j = f // shard
            b = min(n, (j + 1) * shard - offs[t])
            plan.pieces.append(Piece(t, a, b - a, f, j, per_shard[j]))
            per_shard[j] += 1
            a = b
    return plan


# ---------------------------------------------------------------------------
# the exchange


def _check_amax(amax, tensors, spec) -> None:
    """Validate producer maxima for ``tensors`` (see GradientExchange.__call__)."""
    if amax is None:
        return
    if getattr(spec, "normalization", None) is None or spec.normalization.value != "absmax":
        raise UsageError(f"amax applies to absmax specs only, not {spec.label()}")
    dev = tensors[0].device
    if (not isinstance(amax, torch.Tensor) or amax.dtype != torch.float32 or amax.device != dev
            or amax.numel() != len(tensors) or not amax.is_contiguous()):
        raise UsageError(f"amax must be a contiguous float32 tensor of {len(tensors)} maxima on {dev}")
    if dev.type != "cuda":
        raise UsageError("amax needs CUDA tensors")


class _StepRecorder:
    """Records one eager exchange step -- the C-ABI launches with their
    ctypes arguments and the collectives with their tensor views -- so that
    later calls with the same shapes, addresses, stream and workspace replay
    it without rebuilding anything in Python (the eager step's host cost
    otherwise exceeds its GPU time at N > 1).  Arguments equal to the
    recording call's status word are re-pointed at each replay's word."""

    class _Lib:
        def __init__(self, rec):
            self._rec = rec

        def __getattr__(self, name):
            fn = getattr(N.lib, name)

            def call(*args):
                self._rec.ops.append(("lib", fn, list(args)))
                return fn(*args)

            return call

    class _Handle:
        def __init__(self, rec, k, h):
            self._rec, self._k, self._h = rec, k, h

        def wait(self):
            self._rec.ops.append(("wait", self._k))
            return self._h.wait()

    class _Comm:
        def __init__(self, rec, comm):
            self._rec, self._comm = rec, comm
            if not hasattr(comm, "all_gather_async"):
                self.all_gather_async = None  # the step then uses blocking all-gathers

        def world(self):
            return self._comm.world()

        def all_gather(self, out, slot):
            self._rec.ops.append(("ag", out, slot))
            return self._comm.all_gather(out, slot)

        def all_gather_async(self, out, slot):
            k = self._rec.nhandles
            self._rec.nhandles += 1
            self._rec.ops.append(("ag_async", out, slot, k))
            return _StepRecorder._Handle(self._rec, k, self._comm.all_gather_async(out, slot))

        def all_to_all(self, recv, send):
            self._rec.ops.append(("a2a", recv, send))
            return self._comm.all_to_all(recv, send)

    def __init__(self):
        self.ops: list = []
        self.nhandles = 0
        self.status_ptr = None
        self.dyn: list = []  # (op index, arg index) holding the status word

    def finish(self, status_ptr: int) -> None:
        for i, op in enumerate(self.ops):
            if op[0] == "lib":
                for j, a in enumerate(op[2]):
                    if isinstance(a, int) and a == status_ptr:
                        self.dyn.append((i, j))

    def replay(self, comm, status_ptr: int) -> None:
        for i, j in self.dyn:
            self.ops[i][2][j] = status_ptr
        handles: list = [None] * self.nhandles
        for op in self.ops:
            kind = op[0]
            if kind == "lib":
                N.check(op[1](*op[2]))
            elif kind == "ag_async":
                handles[op[3]] = comm.all_gather_async(op[1], op[2])
            elif kind == "wait":
                handles[op[1]].wait()
            elif kind == "ag":
                comm.all_gather(op[1], op[2])
            else:
                comm.all_to_all(op[1], op[2])


class GradientExchange:
    """Compressed all-reduce of a list of float32 tensors (in place by default).

    ``spec``   codec spec (the DP seam default is dynamic-tree/absmax,
               mlp.py:399-411)
    ``mode``   "allgather" or "two_round"
    ``op``     "avg" (data-parallel gradient average) or "sum" (model-parallel
               error-signal sum)
    ``check``  "deferred": the non-finite status of call k is checked at call
               k+1 (or ``synchronize()``) without stalling the stream;
               "sync": checked before returning; "none".
    ``graph``  capture the step (encode, decode, status copy) in a CUDA graph
               per (shapes, input/output addresses) and replay it: one launch
               per step and no host work between the kernels.  Applies on a
               single rank (N = 1); collectives run eagerly.  A graph's
               replays share one host word that counts non-finite replays
               (A8_LAYOUT_STATUS_COUNT), so with deferred checks no report is
               lost: a bad replay raises at the check of that call or of an
               earlier one still pending.
    ``local_fp32``  allgather only: each rank adds its own float32 gradient
               instead of the decode of its own codes -- the paper's "8-bit
               approximation for all incoming GPUs and 32-bit gradients for
               the local GPU".  Ranks then hold different
               (each slightly more accurate) averages.
    Every rank must call it with the same tensor shapes in the same order.
    """

    def __new__(cls, spec=None, *args, **kwargs):
        if cls is GradientExchange and isinstance(spec, str) and spec == ONEBIT:
            return super().__new__(OneBitExchange)  # __init__ runs as OneBitExchange.__init__
        return super().__new__(cls)

    def __init__(self, spec: DataTypeSpec, group=None, mode: str = "allgather", op: str = "avg",
                 check: str = "deferred", codec: Optional[SegmentCodec] = None, comm=None,
                 chunk_elems: int = 8 << 20, max_chunks: int = 8, graph: bool = False,
                 local_fp32: bool = False):
        if mode not in MODES:
            raise UsageError(f"mode must be one of {MODES}, got {mode!r}")
        if op not in OPS:
            raise UsageError(f"op must be one of {OPS}, got {op!r}")
        if check not in ("deferred", "sync", "none"):
            raise UsageError("check must be 'deferred', 'sync' or 'none'")
        if local_fp32 and mode != "allgather":
            raise UsageError("local_fp32 needs mode='allgather'")
        self.spec = spec
        self.cb = build_codebook(spec)
        self.group = group
        self.mode = mode
        self.op = op
        self.check = check
        self.codec = codec or CudaSegmentCodec()
        self.comm = comm or TorchDistComm(group)
        self._plans: dict = {}
        self._bufs: dict = {}
        self._pending = collections.deque()  # (event or None, host status word, call, graph key or None)
        self._ring = None
        self._slot = 0
        self.calls = 0
        self.chunk_elems = int(chunk_elems)  # allgather: elements per pipelined chunk
        self.max_chunks = int(max_chunks)
        self.graph = bool(graph)
        self._graphs: dict = {}
        self._gstream = None
        self._capturing = None  # pinned host status word while capturing
        self._seen: dict = {}  # graph key -> non-finite count already reported
        self._prepared: dict = {}  # eager-step key -> _StepRecorder (CUDA codec only)
        self.local_fp32 = bool(local_fp32)

    # -- distributed context
    def _world(self):
        return self.comm.world()

    def _buffer(self, name: str, nbytes: int, device, dtype=torch.uint8) -> torch.Tensor:
        key = (name, device)
        b = self._bufs.get(key)
        if b is None or b.numel() < nbytes:
            if self._capturing is not None:
                raise UsageError("exchange buffer grew during graph capture")
            b = torch.zeros(nbytes, dtype=dtype, device=device)
            self._bufs[key] = b
            self._graphs.clear()  # captured graphs hold the old buffer's address
            self._prepared.clear()  # and so do recorded steps
        return b[:nbytes]

    # -- status handling
    #
    # The final decode writes the collective status word (OR of every rank's
    # encoder status) straight into pinned host memory (UVA: the kernel
    # stores to the host-mapped word; no device->host copy in the stream).
    # Eager calls take a fresh word from a ring of _RING slots, so every
    # call's status is checked; graph mode bakes one word into each graph.

    _RING = 64
    _PREPARED_MAX = 16  # recorded steps kept (oldest dropped first)

    def _status_word(self, dev) -> torch.Tensor:
        """Where this call's final decode writes its status (uint8[4] view)."""
        if self._capturing is not None:
            return self._capturing
        if self._ring is None:
            pin = dev.type == "cuda"
            self._ring = torch.zeros(self._RING, dtype=torch.int32, pin_memory=pin)
        w = self._ring[self._slot % self._RING:self._slot % self._RING + 1]
        self._slot += 1
        if len(self._pending) >= self._RING - 1:  # the oldest unchecked word is about to be reused
            self._check_one(block=True)
        return w.view(torch.uint8)

    def _collect_status(self, word: torch.Tensor):
        if self._capturing is not None or self.check == "none":
            return
        ev = None
        if word.device.type == "cpu" and torch.cuda.is_available() and word.is_pinned():
            ev = torch.cuda.Event()
            ev.record()
        self._pending.append((ev, word.view(torch.int32), self.calls, None))
        if self.check == "sync":
            self.synchronize()

    def _check_one(self, block: bool) -> bool:
        """Check the oldest pending status; False if it is not ready (non-blocking)."""
        ev, word, call, gkey = self._pending[0]
        if ev is not None:
            if not block and not ev.query():
                return False
            ev.synchronize()
        self._pending.popleft()
        if gkey is not None:  # a graph's word counts its non-finite replays
            count = int(word[0])
            bad = count > self._seen.get(gkey, 0)
            self._seen[gkey] = count
        else:
            w = int(word[0])
            if w & N.A8_STATUS_AMAX_MISMATCH:
                self._pending.clear()
                raise UsageError(f"exchange call {call}: a supplied amax is not max|x| of its tensor")
            bad = bool(w & N.A8_STATUS_NONFINITE)
        if bad:
            self._pending.clear()
            raise InputError(f"exchange call {call}: cannot encode non-finite values (NaN or Inf present)"
                             + (" (or a supplied amax is not max|x|)" if gkey is not None else ""))
        return True

    def synchronize(self) -> None:
        """Wait for every pending exchange status and raise InputError if any
        rank's input held NaN/Inf (codecs.py:251-252)."""
        while self._pending:
            self._check_one(block=True)

    def _poll(self) -> None:
        while self._pending and self._check_one(block=False):
            pass

    # -- main entry
    def __call__(self, tensors: Sequence[torch.Tensor], out: Optional[Sequence[torch.Tensor]] = None,
                 amax: Optional[torch.Tensor] = None):
        """``amax`` (absmax specs): float32 tensor on the inputs' device with
        max|tensors[i]| at [i], written by the kernel that produced the
        tensors (``produce.scale_absmax_``, ``produce.relu_absmax``): the
        encode is then one pass over the inputs (a8_encode_premax).  A wrong
        value raises UsageError at the status check."""
        tensors = list(tensors)
        if not tensors:
            return []
        self._poll()
        dev = tensors[0].device
        _check_amax(amax, tensors, self.spec)
        self._amax = amax
        for t in tensors:
            if t.dtype != torch.float32 or not t.is_contiguous() or t.device != dev:
                raise UsageError("exchange needs contiguous float32 tensors on one device")
        outs = list(out) if out is not None else tensors
        if out is not None:
            if len(outs) != len(tensors):
                raise UsageError(f"out holds {len(outs)} tensors, the call has {len(tensors)}")
            for t, o in zip(tensors, outs):
                if (o.dtype != torch.float32 or not o.is_contiguous() or o.device != dev
                        or o.numel() != t.numel()):
                    raise UsageError("each out tensor must be contiguous float32 on the inputs' device, "
                                     "with as many elements as its input")
        nranks, rank = self._world()
        sizes = tuple(t.numel() for t in tensors)
        key = (sizes, nranks)
        plan = self._plans.get(key)
        if plan is None:
            plan = self._plans[key] = make_plan(sizes, nranks)
        # graphs need launch-inline plans (<= 32 tensors: no host->device plan upload)
        if self.graph and nranks == 1 and dev.type == "cuda" and plan.nseg <= 32:
            self._replay(tensors, outs, plan, nranks, rank, dev)
        elif type(self.codec) is CudaSegmentCodec and dev.type == "cuda":
            self._step_prepared(tensors, outs, plan, nranks, rank, dev)
        else:
            self._step(tensors, outs, plan, nranks, rank, dev)
        self.calls += 1
        return outs

    _amax = None  # the current call's producer maxima (None: the encode computes them)

    def _amax_kw(self) -> dict:
        return {} if self._amax is None else {"amax": self._amax}

    def _step_prepared(self, tensors, outs, plan, nranks, rank, dev):
        """Eager step through a recorded launch list (see _StepRecorder):
        the first call with a key runs normally while recording; later calls
        replay the list.  Steps whose host work is not all launches and
        collectives (two_round on a rank that owns no piece) are not
        recorded."""
        stream = torch.cuda.current_stream(dev).cuda_stream
        key = (plan.sizes, nranks, rank, self.mode, self.op, self.local_fp32, stream,
               workspace_epoch(dev, stream), tuple(t.data_ptr() for t in tensors),
               tuple(o.data_ptr() for o in outs), 0 if self._amax is None else self._amax.data_ptr())
        rec = self._prepared.get(key)
        if rec is not None:
            word = self._status_word(dev)
            rec.replay(self.comm, word.data_ptr())
            self._collect_status(word)
            return
        recordable = self.mode == "allgather" or nranks == 1 or any(p.shard == rank for p in plan.pieces)
        if not recordable:
            self._step(tensors, outs, plan, nranks, rank, dev)
            return
        rec = _StepRecorder()
        codec, comm = self.codec, self.comm
        self.codec._lib = _StepRecorder._Lib(rec)
        self.comm = _StepRecorder._Comm(rec, comm)
        words: list = []
        collect = self._collect_status
        self._collect_status = lambda w: (words.append(w), collect(w))
        try:
            self._step(tensors, outs, plan, nranks, rank, dev)
        finally:
            codec._lib = N.lib
            self.comm = comm
            self._collect_status = collect
        if len(words) == 1 and key[7] == workspace_epoch(dev, stream):
            rec.finish(words[0].data_ptr())
            if len(self._prepared) >= self._PREPARED_MAX:  # callers passing fresh tensors every step
                self._prepared.pop(next(iter(self._prepared)))
            self._prepared[key] = rec

    def _step(self, tensors, outs, plan, nranks, rank, dev):
        if self.mode == "allgather" or nranks == 1:
            self._allgather(tensors, outs, plan, nranks, rank, dev)
        else:
            self._two_round(tensors, outs, plan, nranks, rank, dev)

    def _replay(self, tensors, outs, plan, nranks, rank, dev):
        """Graph mode: the first call with a given (shapes, addresses) runs
        eagerly on a side stream (allocating every buffer and workspace the
        step uses) and captures the step; later calls replay it."""
        key = (plan.sizes, nranks, self.mode, tuple(t.data_ptr() for t in tensors),
               tuple(o.data_ptr() for o in outs), 0 if self._amax is None else self._amax.data_ptr())
        hit = self._graphs.get(key)
        cur = torch.cuda.current_stream(dev)
        if hit is not None and hit[2] != workspace_epoch(dev, self._gstream.cuda_stream):
            # the side stream's workspace was reallocated: the graph holds a freed address
            self._graphs.clear()
            hit = None
        if hit is None:
            if self._gstream is None:
                self._gstream = torch.cuda.Stream(dev)
            s = self._gstream
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                self._step(tensors, outs, plan, nranks, rank, dev)  # this call's result
            cur.wait_stream(s)
            host = torch.zeros(4, dtype=torch.uint8, pin_memory=True)  # this graph's non-finite count
            g = torch.cuda.CUDAGraph()
            self._capturing = host
            try:
                with torch.cuda.graph(g, stream=s):
                    self._step(tensors, outs, plan, nranks, rank, dev)
            finally:
                self._capturing = None
            gkey = object()
            self._seen[gkey] = 0
            self._graphs[key] = (g, host, workspace_epoch(dev, s.cuda_stream), gkey)
            return
        g, host, _, gkey = hit
        g.replay()
        if self.check != "none":
            ev = torch.cuda.Event()
            ev.record(cur)
            self._pending.append((ev, host.view(torch.int32), self.calls, gkey))
            if self.check == "sync":
                self.synchronize()

    def _chunking(self, plan: Plan, nranks: int):
        """K chunk-blocks of C elements for the pipelined all-gather (K = 1
        on one rank or for small buckets).  Cached per plan."""
        key = ("chunks", plan.sizes, nranks)
        hit = self._plans.get(key)
        if hit is None:
            K = 1 if nranks == 1 else int(min(self.max_chunks, max(1, -(-plan.flat // self.chunk_elems))))
            C = round16(-(-plan.flat // K))
            K = -(-plan.flat // C)
            pieces: list = [[] for _ in range(K)]
            for t, n in enumerate(plan.sizes):
                a = 0
                while a < n:
                    f = plan.offs[t] + a
                    j = f // C
                    b = min(n, (j + 1) * C - plan.offs[t])
                    pieces[j].append((t, a, b - a, f))
                    a = b
            hit = self._plans[key] = (K, C, pieces)
        return hit

    def _allgather(self, xs, outs, plan: Plan, nranks, rank, dev):
        """Encode into K chunk-blocks laid out [r0 codes | r0 scales+status |
        r1 codes | ...] (rank stride = C + gap), all-gather each block in
        place, and decode a block's pieces as soon as it has arrived, so the
        decode of block j overlaps the all-gather of block j+1."""
        K, C, pieces = self._chunking(plan, nranks)
        P = C + plan.gap  # one rank's part of a block
        BS = nranks * P  # one block
        gathered = self._buffer("gather", K * BS, dev)
        idx = list(range(plan.nseg))
        mine = rank * P
        self.codec.encode(xs, plan.offs, idx, self.cb, gathered, mine, mine + C, C, BS, BS // 4, K,
                          mine + C + 4 * plan.status_slot, **self._amax_kw())
        status = self._status_word(dev)
        op = 1 if self.op == "avg" else 0
        loc = self.local_fp32
        if nranks == 1:
            self.codec.decode(outs, plan.offs, idx, self.cb, gathered, 0, C, C, BS, BS // 4, P, 1, op,
                              plan.status_slot, 1, status, locals_=xs if loc else None, local_rank=0,
                              status_count=self._capturing is not None)
            self._collect_status(status)
            return
        start = getattr(self.comm, "all_gather_async", None)
        handles = []
        for j in range(K):
            blk = gathered[j * BS:(j + 1) * BS]
            if start is not None:
                handles.append(start(blk, blk[mine:mine + P]))
            else:
                self.comm.all_gather(blk, blk[mine:mine + P])
                handles.append(None)
        for j in range(K):
            if handles[j] is not None:
                handles[j].wait()
            po = [outs[t].view(-1)[a:a + n] for (t, a, n, f) in pieces[j]]
            pl = [xs[t].view(-1)[a:a + n] for (t, a, n, f) in pieces[j]] if loc else None
            self.codec.decode(po, [f for (t, a, n, f) in pieces[j]], [t for (t, a, n, f) in pieces[j]], self.cb,
                              gathered, 0, C, C, BS, BS // 4, P, nranks, op, plan.status_slot, 1,
                              status if j == K - 1 else None, locals_=pl, local_rank=rank)
        self._collect_status(status)

    def _two_round(self, xs, outs, plan: Plan, nranks, rank, dev):
        L = plan.shard
        B = plan.two_round_block()
        sbs = B // 4  # scale areas are B bytes apart
        send = self._buffer("send", nranks * B, dev)
        recv = self._buffer("recv", nranks * B, dev)
        idx = list(range(plan.nseg))
        # round 1: per-tensor encode straight into the N send blocks
        self.codec.encode(xs, plan.offs, idx, self.cb, send, 0, L, L, B, sbs, nranks,
                          L + 4 * plan.status_slot, **self._amax_kw())
        self.comm.all_to_all(recv, send)
        # decode-average the N contributions to my shard
        mine = [p for p in plan.pieces if p.shard == rank]
        shard_buf = self._buffer("shard", max(L, 16) * 4, dev).view(torch.float32)
        pouts = [shard_buf[p.flat - rank * L: p.flat - rank * L + p.n] for p in mine]
        poffs = [p.flat - rank * L for p in mine]
        status1 = self._buffer("status1", 4, dev)
        self.codec.decode(pouts, poffs, [p.tensor for p in mine], self.cb, recv, 0, L, L, B, 0, B,
                          nranks, 1 if self.op == "avg" else 0, plan.status_slot, 1, status1)
        # round-2 blocks: chunk_elems of gathered data per block, as for allgather
        K2 = 1 if nranks == 1 else int(min(self.max_chunks, max(1, -(-L // max(16, self.chunk_elems // nranks)))))
        if K2 > 1:
            self._two_round_pipelined_r2(outs, plan, nranks, rank, dev, mine, pouts, poffs, status1, K2)
            return
        # round 2: re-encode my shard, one scale per piece, into my gather slot
        gathered = self._buffer("gather2", nranks * B, dev)
        slot = rank * B
        status_off = slot + L + 4 * plan.status_slot
        if mine:
            # round-1 status is chained into the round-2 word by the kernel
            self.codec.encode(pouts, poffs, [p.idx for p in mine], self.cb, gathered, slot,
                              slot + L, L, B, 0, 1, status_off, status_in=status1)
        else:
            gathered[status_off:status_off + 4].copy_(status1)
        self.comm.all_gather(gathered, gathered[slot:slot + B])
        # final decode of every piece straight into the outputs
        fouts, foffs, fidx = [], [], []
        for p in plan.pieces:
            fouts.append(outs[p.tensor].view(-1)[p.start:p.start + p.n])
            foffs.append(p.flat)
            fidx.append(p.idx)
        status = self._status_word(dev)
        self.codec.decode(fouts, foffs, fidx, self.cb, gathered, 0, L, L, B, sbs, 0, 1, 0,
                          plan.status_slot, nranks, status)
        self._collect_status(status)


    def _two_round_pipelined_r2(self, outs, plan: Plan, nranks, rank, dev, mine, pouts, poffs, status1, K2):
        """Round 2 of two_round with the all-gather split into K2 blocks: block
        k holds chunk k (Ck elements) of every rank's shard, laid out
        [r0 codes | r0 scales+status | r1 ...].  One re-encode launch writes
        all K2 blocks of my shard (per-piece scales, as for K2 = 1), then
        block k is all-gathered in place while block k-1 is decoded.  The
        pieces and scales are those of the unpipelined round 2, so the result
        does not depend on K2."""
        L = plan.shard
        Ck = round16(-(-L // K2))
        K2 = -(-L // Ck)
        P = Ck + plan.gap  # one rank's part of a block
        BS = nranks * P
        gathered = self._buffer("gather2p", K2 * BS, dev)
        slot = rank * P
        status_off = slot + Ck + 4 * plan.status_slot
        if mine:
            self.codec.encode(pouts, poffs, [p.idx for p in mine], self.cb, gathered, slot, slot + Ck, Ck, BS,
                              BS // 4, K2, status_off, status_in=status1)
        else:
            for k in range(K2):
                gathered[k * BS + status_off:k * BS + status_off + 4].copy_(status1)
        start = getattr(self.comm, "all_gather_async", None)
        handles = []
        for k in range(K2):
            blk = gathered[k * BS:(k + 1) * BS]
            if start is not None:
                handles.append(start(blk, blk[slot:slot + P]))
            else:
                self.comm.all_gather(blk, blk[slot:slot + P])
                handles.append(None)
        # pieces of every rank's shard, cut at chunk boundaries
        sub: list = [[] for _ in range(K2)]
        for p in plan.pieces:
            o0 = p.flat - p.shard * L  # piece start inside its shard
            a = o0
            while a < o0 + p.n:
                k = a // Ck
                b = min(o0 + p.n, (k + 1) * Ck)
                view = outs[p.tensor].view(-1)[p.start + (a - o0):p.start + (b - o0)]
                sub[k].append((view, p.shard * Ck + (a - k * Ck), p.idx))
                a = b
        status = self._status_word(dev)
        for k in range(K2):
            if handles[k] is not None:
                handles[k].wait()
            self.codec.decode([v for v, f, i in sub[k]], [f for v, f, i in sub[k]], [i for v, f, i in sub[k]],
                              self.cb, gathered, k * BS, k * BS + Ck, Ck, P, P // 4, 0, 1, 0,
                              plan.status_slot, nranks, status if k == K2 - 1 else None)
        self._collect_status(status)


class OneBitExchange(GradientExchange):
    """1-bit error-feedback gradient exchange: ``GradientExchange("onebit")``.

    The reference's 1-bit data-parallel seam (mlp.py:313-321) quantizes every
    gradient with ``onebit_quantize`` and a residual carried per tensor
    across steps (codecs.py:291-348), then trains on ``onebit_decode``.
    Across N ranks: every rank quantizes each tensor with its own residual
    (a float64 tensor kept on the device, one per tensor position), the
    packed bits and the two float32 levels of every tensor travel in one slab
    [bits (each tensor padded to 16 B) | levels | status words], the slabs
    are all-gathered with NCCL, and one launch decodes, sums in rank order in
    float32 and divides by N (a8_onebit_reduce).  32x less payload than
    float32 on the wire.  Oracle: oracle.exchange_onebit.

    Residuals are keyed by (position, numel); ``reset()`` drops them.
    Non-finite input raises ``InputError`` (on every rank) and leaves every
    residual untouched.  allgather only; ``graph`` is not supported.
    """

    def __init__(self, spec=ONEBIT, group=None, mode: str = "allgather", op: str = "avg", check: str = "deferred",
                 codec: Optional[SegmentCodec] = None, comm=None, **unused):
        if spec != ONEBIT:
            raise UsageError(f"OneBitExchange needs spec={ONEBIT!r}")
        if mode != "allgather":
            raise UsageError("the 1-bit exchange is an all-gather (mode='allgather')")
        if op not in OPS:
            raise UsageError(f"op must be one of {OPS}, got {op!r}")
        if check not in ("deferred", "sync", "none"):
            raise UsageError("check must be 'deferred', 'sync' or 'none'")
        if unused.get("graph") or unused.get("local_fp32"):
            raise UsageError("graph / local_fp32 are not supported by the 1-bit exchange")
        self.spec = ONEBIT
        self.cb = None
        self.group = group
        self.mode = mode
        self.op = op
        self.check = check
        self.codec = codec or CudaSegmentCodec()
        self.comm = comm or TorchDistComm(group)
        self._plans: dict = {}
        self._bufs: dict = {}
        self._pending = collections.deque()
        self._ring = None
        self._slot = 0
        self.calls = 0
        self.graph = False
        self._graphs: dict = {}
        self._gstream = None
        self._capturing = None
        self._seen: dict = {}
        self._prepared: dict = {}
        self.local_fp32 = False
        self.residuals: dict = {}  # (position, numel) -> float64 residual tensor

    def reset(self) -> None:
        self.residuals.clear()

    @staticmethod
    def layout(sizes):
        """(bit offsets, levels offset, status offset, slab bytes) of one rank's slab."""
        offs, pos = [], 0
        for n in sizes:
            offs.append(pos)
            pos += round16(-(-int(n) // 8))
        lev = pos
        st = lev + 8 * len(sizes)
        return offs, lev, st, round16(st + 4 * len(sizes))

    def __call__(self, tensors: Sequence[torch.Tensor], out: Optional[Sequence[torch.Tensor]] = None):
        tensors = list(tensors)
        if not tensors:
            return []
        self._poll()
        dev = tensors[0].device
        for t in tensors:
            if t.dtype not in (torch.float32, torch.float64) or not t.is_contiguous() or t.device != dev:
                raise UsageError("the 1-bit exchange needs contiguous float32/float64 tensors on one device")
        outs = list(out) if out is not None else tensors
        for t, o in zip(tensors, outs):
            if o.dtype != torch.float32 or not o.is_contiguous() or o.device != dev or o.numel() != t.numel():
                raise UsageError("each out tensor must be contiguous float32 on the inputs' device, "
                                 "with as many elements as its input")
        if len(outs) != len(tensors):
            raise UsageError(f"out holds {len(outs)} tensors, the call has {len(tensors)}")
        if any(t.dtype != torch.float32 for t in outs) and out is None:
            raise UsageError("in-place 1-bit exchange needs float32 tensors (pass out= for float64 input)")
        nranks, rank = self._world()
        sizes = tuple(t.numel() for t in tensors)
        offs, lev, st, P = self.layout(sizes)
        buf = self._buffer("onebit", nranks * P, dev)
        mine = rank * P
        res = []
        for i, t in enumerate(tensors):
            key = (i, t.numel())
            r = self.residuals.get(key)
            if r is None:
                r = self.residuals[key] = torch.zeros(t.numel(), dtype=torch.float64, device=dev)
            res.append(r)
        # each rank's residual follows its own onebit_quantize exactly: updated
        # iff its own input is finite (the kernel leaves it untouched otherwise,
        # codecs.py:317-318); a non-finite input on any rank raises InputError
        # on every rank (the status words travel in the slabs)
        many = getattr(self.codec, "onebit_quantize_many", None)
        if many is not None:  # all tensors in two launches
            many([t.reshape(-1) for t in tensors], res, buf, [mine + o for o in offs],
                 [mine + lev + 8 * i for i in range(len(tensors))], [mine + st + 4 * i for i in range(len(tensors))])
        else:
            for i, t in enumerate(tensors):
                self.codec.onebit_quantize(t.reshape(-1), res[i], buf, mine + offs[i], mine + lev + 8 * i,
                                           mine + st + 4 * i)
        if nranks > 1:
            self.comm.all_gather(buf, buf[mine:mine + P])
        status = self._status_word(dev)
        self.codec.onebit_reduce([o.reshape(-1) for o in outs], offs, buf, P, lev, st, nranks,
                                 1 if self.op == "avg" else 0, status)
        self._collect_status(status)
        self.calls += 1
        return outs


# ---------------------------------------------------------------------------
# the exchange over NVLink peer memory: the decode reads the other GPUs'
# codes directly (no collective, no gathered copy in HBM)


class PeerTransport:
    """Buffers every rank of the group can read directly, plus a
    stream-ordered barrier.  ``buffer`` returns this rank's buffer and the
    device base address of every rank's buffer of that name."""

    def world(self):
        raise NotImplementedError

    def buffer(self, name: str, nbytes: int, device):
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError


class SymmetricMemoryTransport(PeerTransport):
    """torch.distributed._symmetric_memory on the NCCL group: buffers mapped
    into every GPU's address space over NVLink (``buffer_ptrs``), and its
    device-side barrier on the current stream."""

    def __init__(self, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self._symm = symm_mem
        self.group = group if group is not None else dist.group.WORLD
        self._bufs: dict = {}
        self._hdl = None

    def world(self):
        return dist.get_world_size(self.group), dist.get_rank(self.group)

    def buffer(self, name, nbytes, device):
        hit = self._bufs.get(name)
        if hit is None or hit[0].numel() < nbytes:
            t = self._symm.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
            t.zero_()
            hdl = self._symm.rendezvous(t, self.group)
            hit = self._bufs[name] = (t, [int(p) for p in hdl.buffer_ptrs], hdl)
            self._hdl = hdl
        return hit[0][:nbytes], hit[1]

    def barrier(self) -> None:
        self._hdl.barrier(channel=0)


class PeerExchange(GradientExchange):
    """``GradientExchange`` whose data movement is the decode kernel itself
    reading the peers' slabs over NVLink (``a8_decode_peers``): each rank
    encodes into its own slab of a peer-mapped buffer, one barrier, and
    the fused decode-sum(-average) pulls every rank's codes and scales from
    their GPUs.  Same numerics and oracles as the NCCL path.

    ``allgather``: slab [codes | scales | status]; one barrier per call
    (the slabs are double-buffered, so the next call's barrier also orders
    the peers' reads before the buffer is rewritten).
    ``two_round``: round 1 reads, from every peer, the block of its codes
    destined to this rank's shard (the all-to-all becomes peer loads inside
    the decode); the averaged shard is re-encoded into a second slab; after
    a second barrier, round 2 decodes every shard from its owner's slab.
    """

    def __init__(self, spec: DataTypeSpec, transport: PeerTransport, mode: str = "allgather", op: str = "avg",
                 check: str = "deferred", codec: Optional[SegmentCodec] = None):
        super().__init__(spec, None, mode, op, check, codec)
        self.transport = transport
        self.comm = transport  # world()

    def __call__(self, tensors: Sequence[torch.Tensor], out: Optional[Sequence[torch.Tensor]] = None,
                 amax: Optional[torch.Tensor] = None):
        tensors = list(tensors)
        if not tensors:
            return []
        self._poll()
        dev = tensors[0].device
        for t in tensors:
            if t.dtype != torch.float32 or not t.is_contiguous() or t.device != dev:
                raise UsageError("exchange needs contiguous float32 tensors on one device")
        _check_amax(amax, tensors, self.spec)
        self._amax = amax
        outs = list(out) if out is not None else tensors
        if len(outs) != len(tensors) or any(o.dtype != torch.float32 or not o.is_contiguous() or o.device != dev
                                            or o.numel() != t.numel() for t, o in zip(tensors, outs)):
            raise UsageError("each out tensor must be contiguous float32 on the inputs' device, "
                             "with as many elements as its input")
        nranks, rank = self.transport.world()
        sizes = tuple(t.numel() for t in tensors)
        plan = self._plans.get((sizes, nranks))
        if plan is None:
            plan = self._plans[(sizes, nranks)] = make_plan(sizes, nranks)
        par = self.calls & 1
        if self.mode == "allgather" or nranks == 1:
            self._peer_allgather(tensors, outs, plan, nranks, rank, dev, par)
        else:
            self._peer_two_round(tensors, outs, plan, nranks, rank, dev, par)
        self.calls += 1
        return outs

    def _peer_allgather(self, xs, outs, plan, nranks, rank, dev, par):
        C = plan.flat
        P = plan.allgather_block()
        slab, ptrs = self.transport.buffer(f"ag{par}", P, dev)
        idx = list(range(plan.nseg))
        self.codec.encode(xs, plan.offs, idx, self.cb, slab, 0, C, C, C, 0, 1, C + 4 * plan.status_slot,
                          **self._amax_kw())
        self.transport.barrier()
        status = self._status_word(dev)
        self.codec.decode_peers(outs, plan.offs, idx, self.cb, 0, C, C, C, 0, ptrs[:nranks],
                                1 if self.op == "avg" else 0, plan.status_slot, 1, status)
        self._collect_status(status)

    def _peer_two_round(self, xs, outs, plan, nranks, rank, dev, par):
        L = plan.shard
        B = plan.two_round_block()
        sbs = B // 4
        send, sptrs = self.transport.buffer(f"tr_send{par}", nranks * B, dev)
        idx = list(range(plan.nseg))
        # round 1: per-tensor encode into the N destination blocks of my slab
        self.codec.encode(xs, plan.offs, idx, self.cb, send, 0, L, L, B, sbs, nranks, L + 4 * plan.status_slot,
                          **self._amax_kw())
        self.transport.barrier()
        mine = [p for p in plan.pieces if p.shard == rank]
        shard_buf = self._buffer("shard", max(L, 16) * 4, dev).view(torch.float32)
        pouts = [shard_buf[p.flat - rank * L: p.flat - rank * L + p.n] for p in mine]
        poffs = [p.flat - rank * L for p in mine]
        status1 = self._buffer("status1", 4, dev)
        # rank r's block for my shard sits at its slab + rank * B
        bases = [b + rank * B for b in sptrs[:nranks]]
        self.codec.decode_peers(pouts, poffs, [p.tensor for p in mine], self.cb, 0, L, L, B, 0,
                                bases, 1 if self.op == "avg" else 0, plan.status_slot, 1, status1)
        # round 2: my averaged shard, one scale per piece, into my gather slab
        gath, gptrs = self.transport.buffer(f"tr_gather{par}", B, dev)
        status_off = L + 4 * plan.status_slot
        if mine:
            self.codec.encode(pouts, poffs, [p.idx for p in mine], self.cb, gath, 0, L, L, B, 0, 1, status_off,
                              status_in=status1)
        else:
            gath[status_off:status_off + 4].copy_(status1)
        self.transport.barrier()
        sts = self._buffer("status2", 4 * nranks, dev).view(torch.int32)
        for j in range(nranks):
            pj = [p for p in plan.pieces if p.shard == j]
            self.codec.decode_peers([outs[p.tensor].view(-1)[p.start:p.start + p.n] for p in pj],
                                    [p.flat - j * L for p in pj], [p.idx for p in pj], self.cb, 0, L, L, B, 0,
                                    [gptrs[j]], 0, plan.status_slot, 1, sts[j:j + 1].view(torch.uint8))
        status = self._status_word(dev)
        status.view(torch.int32).copy_(sts.amax().view(1), non_blocking=True)
        self._collect_status(status)


def exchange(tensors, spec: DataTypeSpec, group=None, mode: str = "allgather", op: str = "avg"):
    """One-shot functional form of ``GradientExchange`` (check="sync")."""
    return GradientExchange(spec, group, mode, op, check="sync")(tensors)


class CompressedAllGather:
    """8-bit all-gather (concatenation, no reduction) of one float32 tensor
    per rank: the model-parallel activation seam (mlp.py:208-215, "the
    activation shipped to the next device").  Each rank encodes its shard
    with its own absmax scale into its slab, the slabs are all-gathered, and
    one decode launch writes every rank's decoded shard into ``out[r]``."""

    def __init__(self, spec: DataTypeSpec, group=None, codec: Optional[SegmentCodec] = None, comm=None):
        self.spec = spec
        self.cb = build_codebook(spec)
        self.codec = codec or CudaSegmentCodec()
        self.comm = comm or TorchDistComm(group)
        self._bufs: dict = {}

    def __call__(self, shard: torch.Tensor, out: Optional[Sequence[torch.Tensor]] = None,
                 amax: Optional[torch.Tensor] = None):
        """``amax``: max|shard| from its producer (float32, 1 element), see
        GradientExchange.__call__."""
        if shard.dtype != torch.float32 or not shard.is_contiguous():
            raise UsageError("all-gather needs a contiguous float32 tensor")
        _check_amax(amax, [shard], self.spec)
        nranks, rank = self.comm.world()
        dev = shard.device
        n = shard.numel()
        plan = make_plan((n,), 1)
        B = plan.allgather_block()
        key = (n, nranks, dev)
        if key not in self._bufs:
            self._bufs[key] = (torch.zeros(nranks * B, dtype=torch.uint8, device=dev),
                               torch.zeros(1, dtype=torch.int32, device=dev))
        slab, status = self._bufs[key]
        self.codec.encode([shard], [0], [0], self.cb, slab, rank * B, rank * B + plan.flat, plan.flat,
                          plan.flat, 0, 1, rank * B + plan.flat + 4 * plan.status_slot,
                          **({} if amax is None else {"amax": amax}))
        if nranks > 1:
            self.comm.all_gather(slab, slab[rank * B:(rank + 1) * B])
        outs = list(out) if out is not None else [torch.empty_like(shard) for _ in range(nranks)]
        # rank j's shard is segment j of a layout whose blocks are the slabs
        flat_offs = [j * plan.flat for j in range(nranks)]
        self.codec.decode(outs, flat_offs, [0] * nranks, self.cb, slab, 0, plan.flat, plan.flat, B, B // 4,
                          0, 1, 0, plan.status_slot, nranks, status)
        st = int(status.cpu()[0])
        if st & N.A8_STATUS_AMAX_MISMATCH:
            raise UsageError("the supplied amax is not max|shard|")
        if st & N.A8_STATUS_NONFINITE:
            raise InputError("cannot encode non-finite values (NaN or Inf present)")
        return outs


class LocalExchange:
    """The allgather exchange among N replicas that live in ONE process on
    one device (e.g. several model replicas per GPU): every replica's tensors
    are encoded into its slab of one buffer -- the slabs are then already
    "gathered" -- and one decode-sum(-average) launch writes the result for
    all replicas.  Same kernels, slab layout and numerics as
    ``GradientExchange(mode="allgather")`` with N ranks."""

    def __init__(self, spec: DataTypeSpec, op: str = "avg", codec: Optional[SegmentCodec] = None):
        if op not in OPS:
            raise UsageError(f"op must be one of {OPS}, got {op!r}")
        self.spec = spec
        self.cb = build_codebook(spec)
        self.op = op
        self.codec = codec or CudaSegmentCodec()
        self._bufs: dict = {}

    def __call__(self, per_replica: Sequence[Sequence[torch.Tensor]], out: Optional[Sequence[torch.Tensor]] = None):
        """per_replica[r] = replica r's tensors (same shapes for every r).
        Returns (or fills ``out`` with) one averaged/summed list."""
        nranks = len(per_replica)
        if nranks < 1:
            raise UsageError("need at least one replica")
        first = list(per_replica[0])
        sizes = tuple(t.numel() for t in first)
        for rep in per_replica:
            if tuple(t.numel() for t in rep) != sizes:
                raise UsageError("every replica must hold tensors of the same sizes")
            for t in rep:
                if t.dtype != torch.float32 or not t.is_contiguous() or t.device != first[0].device:
                    raise UsageError("exchange needs contiguous float32 tensors on one device")
        dev = first[0].device
        plan = make_plan(sizes, 1)
        B = plan.allgather_block()
        key = (sizes, nranks, dev)
        buf = self._bufs.get(key)
        if buf is None:
            buf = self._bufs[key] = (torch.zeros(nranks * B, dtype=torch.uint8, device=dev),
                                     torch.zeros(1, dtype=torch.int32, device=dev))
        slab, status = buf
        idx = list(range(plan.nseg))
        for r, rep in enumerate(per_replica):
            self.codec.encode(list(rep), plan.offs, idx, self.cb, slab, r * B, r * B + plan.flat,
                              plan.flat, plan.flat, 0, 1, r * B + plan.flat + 4 * plan.status_slot)
        outs = list(out) if out is not None else [torch.empty_like(t) for t in first]
        self.codec.decode(outs, plan.offs, idx, self.cb, slab, 0, plan.flat, plan.flat, plan.flat, 0, B,
                          nranks, 1 if self.op == "avg" else 0, plan.status_slot, 1, status)
        if int(status.cpu()[0]) & N.A8_STATUS_NONFINITE:
            raise InputError("cannot encode non-finite values (NaN or Inf present)")
        return outs


# ---------------------------------------------------------------------------
# DDP communication hook


class DDPHookState:
    """State of ``a8_comm_hook``: one ``GradientExchange`` (op="avg") shared by
    the buckets of a ``DistributedDataParallel`` model.  ``codec`` / ``comm``
    as for ``GradientExchange`` (tests inject CPU stand-ins)."""

    def __init__(self, spec, group=None, mode: str = "allgather", codec: Optional[SegmentCodec] = None,
                 comm=None, check: str = "deferred"):
        # spec: a DataTypeSpec (8-bit) or "onebit" (1-bit error feedback, one residual per parameter view)
        self.exchange = GradientExchange(spec, group, mode, "avg", check=check, codec=codec, comm=comm)


def a8_comm_hook(state, bucket):
    """``DistributedDataParallel.register_comm_hook(state, a8_comm_hook)``:
    the bucket's per-parameter gradient views are exchanged 8-bit with one
    scale per parameter (the reference's per-tensor seam, mlp.py:367-369)."""
    grads = [g for g in bucket.gradients()]
    state.exchange(grads)
    fut: torch.futures.Future = torch.futures.Future()
    fut.set_result(bucket.buffer())
    return fut


# DDP checks the hook's annotations by identity (not as strings, which is what
# `from __future__ import annotations` would leave here)
a8_comm_hook.__annotations__ = {"state": DDPHookState, "bucket": dist.GradBucket,
                                "return": torch.futures.Future[torch.Tensor]}
