"""Benchmark of the 8-bit approximation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--mode allgather|two_round] [--no-cpu] [--no-sweep] [--eager]

Metric (BASELINE.json): "8-bit codec GB/s vs HBM peak; compressed grad
exchange fp32-equiv GB/s @1/2/4/8 GPU".  One step = one compressed exchange
of a full synthetic gradient set per rank (BASELINE config 3: AlexNet-sized,
61,100,840 float32 parameters in 16 tensors, N(0, 1e-3), seed 1000+16*rank+t):
encode (per-tensor absmax) -> 8-bit all-gather over NCCL (N > 1) ->
fused decode-sum-average.  At N = 1 the step is the codec round trip.

value      = N * 4 B * 61,100,840 / step time   (fp32-equivalent GB/s, whole job)
roofline   = the dominant kernel's algorithmic bytes / its CUDA-event time,
             against the measured HBM copy bandwidth (MEASURED_PEAKS.json)
e2e        = the same exchange through the public API with host buffers:
             pinned H2D of the gradients + exchange + D2H of the averaged
             result, all inside the timed region
cpu_baseline / --impl reference = the reference algorithm on the host cores
             (the oracle port of approx8.codecs; NumPy, all threads)

Inputs (244 MB per rank) exceed the 126 MB L2, so no flush is needed between
steps.  Timing: CUDA events on the launching stream, W warm-up steps, barrier
+ synchronize around the K timed steps, max over ranks.  The timed steps run
the product exchange (at N = 1 its CUDA graph: encode + decode, no event
nodes).  The per-kernel durations behind `roofline` come from K further
steps of an identical exchange whose codec calls are wrapped in CUDA events
on the launching stream (captured into its graph at N = 1 and read after
each replay): event-record nodes between the kernels cost ~15 us per step,
so they stay out of the timed region.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "8-bit codec GB/s vs HBM peak; compressed grad exchange fp32-equiv GB/s @1/2/4/8 GPU"
ALEXNET = [(64, 3, 11, 11), (64,), (192, 64, 5, 5), (192,), (384, 192, 3, 3), (384,),
           (256, 384, 3, 3), (256,), (256, 256, 3, 3), (256,), (4096, 9216), (4096,),
           (4096, 4096), (4096,), (1000, 4096), (1000,)]
SIGMA = 1e-3
SPEC_LABEL = "dynamic-tree/absmax"


def alexnet_grads(rank: int):
    """Config 3 synthetic gradients: one N(0, sigma) draw per
    tensor, seed 1000 + 16*rank + t, float32 (errorbench.sample recipe)."""
    out = []
    for t, shape in enumerate(ALEXNET):
        rng = np.random.default_rng(1000 + 16 * rank + t)
        out.append(rng.normal(0.0, SIGMA, int(np.prod(shape))).astype(np.float32).reshape(shape))
    return out


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the reference's own CPU implementation


def reference_codec():
    """(roundtrip function, kind): the UNMODIFIED reference ``approx8`` from
    baseline/_ref (tools/install_reference.sh) when it is importable there,
    else the oracle port of its algorithm (oracle/approx8_oracle.py)."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "approx8" / "codecs.py").exists():
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        try:
            from approx8 import DataTypeSpec, roundtrip  # noqa: F401

            spec = DataTypeSpec("dynamic-tree", "absmax")
            return (lambda x: roundtrip(x, spec)), "reference"
        except Exception:  # noqa: BLE001  (fall back to the port)
            pass
    from oracle import approx8_oracle as O

    return (lambda x: O.roundtrip(x, "dynamic-tree", "absmax")), "port"


def cpu_reference_step(per_rank, nranks: int, threads: int, rt):
    """One exchange step of the reference algorithm: every rank's tensors
    round-trip through encode_buffer/decode_buffer (codecs.py:244-288) and
    are averaged in rank order in float32 (the composed exchange oracle,
    SURVEY 8(c)); tensors (and ranks) are spread over the host threads, the
    largest first, as the reference's own thread model runs independent
    buffers (errorbench.py:130-139, 172)."""
    jobs = sorted(((r, i) for r in range(nranks) for i in range(len(per_rank[r]))),
                  key=lambda ri: -per_rank[ri[0]][ri[1]].size)
    out: dict = {}
    with cf.ThreadPoolExecutor(max_workers=threads) as pool:
        for (r, i), d in zip(jobs, pool.map(lambda ri: rt(per_rank[ri[0]][ri[1]]), jobs)):
            out[(r, i)] = d
    for i in range(len(per_rank[0])):
        acc = out[(0, i)]
        for r in range(1, nranks):
            acc = acc + out[(r, i)]
        if nranks > 1:
            acc = acc / np.float32(nranks)
    return out


def single_core_rate(rt, elems: int = 1 << 22):
    """Reference round-trip throughput of ONE host core (fp32 GB/s), on one
    2^22-element tensor of the workload's distribution."""
    x = np.random.default_rng(1000).normal(0.0, SIGMA, elems).astype(np.float32)
    rt(x)
    t0 = time.perf_counter()
    rt(x)
    return 4.0 * elems / (time.perf_counter() - t0) / 1e9


def run_reference(args, nranks, rank):
    """--impl reference: the reference's CPU implementation on the SAME
    workload as the B200 arm (config 3: all 16 AlexNet tensors of every rank,
    61,100,840 elements each), all host threads; rank 0 only."""
    if rank != 0:
        return
    rt, kind = reference_codec()
    threads = os.cpu_count() or 1
    per_rank = [alexnet_grads(r) for r in range(nranks)]
    n = sum(g.size for g in per_rank[0])
    warm = min(args.warmup, 1)  # each step is the full workload (seconds): one warm-up pass suffices
    for _ in range(warm):
        cpu_reference_step(per_rank, nranks, threads, rt)
    steps = max(1, min(args.steps, int(os.environ.get("A8_REF_MAX_STEPS", "5"))))
    t0 = time.perf_counter()
    for _ in range(steps):
        cpu_reference_step(per_rank, nranks, threads, rt)
    dt = (time.perf_counter() - t0) / steps
    value = nranks * 4.0 * n / dt / 1e9
    one = single_core_rate(rt)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": nranks,
        "steps": steps, "warmup": warm, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args, nranks),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": kind,
                         "sample": f"the full workload every step: {nranks} rank(s) x 16 AlexNet tensors "
                                   f"({n} elements per rank) N(0,{SIGMA}), "
                                   + ("unmodified approx8 (baseline/_ref) roundtrip" if kind == "reference"
                                      else "oracle port of approx8.codecs roundtrip")
                                   + " per tensor + rank-ordered float32 average; tensors over the threads",
                         "single_core": {"value": one, "unit": "GB/s", "cores": 1,
                                         "sample": "one 2^22-element tensor, one round trip"},
                         "lscpu_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.steps != steps:
        line["note"] = f"timed {steps} full-workload steps (A8_REF_MAX_STEPS) of the requested {args.steps}"
    print(json.dumps(line), flush=True)


def workload_config(args, nranks):
    n = sum(int(np.prod(s)) for s in ALEXNET)
    return {"workload": "C3 AlexNet-sized synthetic gradient exchange", "elements_per_rank": n,
            "tensors": len(ALEXNET), "spec": SPEC_LABEL, "scale": "per-tensor absmax",
            "mode": args.mode if nranks > 1 else "roundtrip (N=1)", "op": "avg",
            "parallelism": f"dp{nranks}", "l2": "inputs 244 MB/rank > 126 MB L2, no flush"}


# ---------------------------------------------------------------------------
# N > 1: parity of the exchange this run measured, and the fp32 NCCL legs

PARITY_SIZES = [(int(np.prod(s)) if np.prod(s) <= 40000 else 40000 + 37 * t,) for t, s in enumerate(ALEXNET)]


def parity_small(A, dist, mode, nranks, rank, dev):
    """The same GradientExchange path as the timed step (same mode, op, NCCL
    collectives, pipelined chunk blocks) on reduced AlexNet-shaped tensors,
    against the composed oracle (oracle/approx8_oracle.py),
    bit for bit.  Every rank regenerates every rank's (seeded) inputs."""
    from oracle import approx8_oracle as O

    def grads(r):
        out = []
        for t, (n,) in enumerate(PARITY_SIZES):
            rng = np.random.default_rng(1000 + 16 * r + t)
            out.append(rng.normal(0.0, SIGMA, n).astype(np.float32))
        return out

    per = [grads(r) for r in range(nranks)]
    want = (O.exchange_allgather(per, "dynamic-tree", "absmax", op="avg") if mode == "allgather"
            else O.exchange_two_round(per, "dynamic-tree", "absmax", op="avg"))
    ex = A.GradientExchange(A.parse_spec(SPEC_LABEL), mode=mode, op="avg", check="sync", chunk_elems=1 << 16)
    mine = [__import__("torch").from_numpy(g).to(dev) for g in per[rank]]
    ex(mine)
    ok = all(m.cpu().numpy().tobytes() == w.astype(np.float32).tobytes() for m, w in zip(mine, want))
    blocks = ex._chunking(ex._plans[(tuple(g.size for g in per[rank]), nranks)], nranks)[0] if mode == "allgather" else None
    return ok, blocks


def outputs_agree(dist, outs, nranks):
    """sha256 of this rank's output bytes, compared across ranks (allgather
    and two_round both leave identical averages on every rank)."""
    import hashlib

    h = hashlib.sha256()
    for o in outs:
        h.update(o.cpu().numpy().tobytes())
    digests = [None] * nranks
    dist.all_gather_object(digests, h.hexdigest())
    return len(set(digests)) == 1, digests[0][:16]


def nccl_leg(dist, algo, n, steps, rank, nranks, local_rank, child_args=None):
    """fp32 NCCL all-reduce of an n-float buffer, in child processes (one per
    rank) with NCCL_ALGO=<algo> (or NCCL's default choice), since NCCL reads
    its tuning environment once per process.  NCCL_DEBUG output is scanned
    for the algorithm it chose."""
    import socket

    port = [0]
    if rank == 0:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port[0] = sk.getsockname()[1]
    dist.broadcast_object_list(port, src=0)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port[0]), RANK=str(rank),
               WORLD_SIZE=str(nranks), LOCAL_RANK=str(local_rank), NCCL_DEBUG="INFO",
               NCCL_DEBUG_SUBSYS="INIT,TUNING,COLL")
    env.pop("NCCL_ALGO", None)
    if algo != "default":
        env["NCCL_ALGO"] = algo
    try:
        cmd = child_args or ["--nccl-leg", str(n)]
        res = subprocess.run([sys.executable, str(Path(__file__).resolve()), *cmd, "--steps", str(steps)],
                             env=env, capture_output=True, text=True, timeout=300)
    except subprocess.TimeoutExpired:
        return {"algo_requested": algo, "error": "timed out after 300 s"} if rank == 0 else None
    out = None
    for line in res.stdout.splitlines():
        if line.startswith("{"):
            out = json.loads(line)
    seen = sorted({ln.split("NCCL INFO", 1)[1].strip()[:120] for ln in (res.stdout + res.stderr).splitlines()
                   if "NCCL INFO" in ln and any(k in ln for k in ("Algo", "NVLS", "algorithm"))})[:6]
    if out is not None:
        out["algo_requested"] = algo
        out["nccl_debug_algo_lines"] = seen
    elif rank == 0:
        out = {"algo_requested": algo, "error": (res.stderr or "")[-300:]}
    return out


def nccl_leg_child(n, steps):
    """--nccl-leg: the child side of nccl_leg (torchrun-style env)."""
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idx = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    torch.cuda.set_device(idx)
    dist.init_process_group("nccl", device_id=torch.device("cuda", idx))
    buf = torch.randn(n, device="cuda")
    for _ in range(3):
        dist.all_reduce(buf)
    torch.cuda.synchronize()
    dist.barrier(device_ids=[idx])
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(steps):
        dist.all_reduce(buf)
    a1.record()
    torch.cuda.synchronize()
    t = torch.tensor([a0.elapsed_time(a1) / steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item())
        print(json.dumps({"value": world * 4.0 * n / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                          "busbw_GBps": 2 * (world - 1) / world * 4.0 * n / (ms * 1e-3) / 1e9}), flush=True)
    dist.destroy_process_group()


def peer_leg_child(mode, steps):
    """--peer-leg MODE: the C3 exchange through PeerExchange (the decode reads
    the peers' slabs over NVLink, torch symmetric memory) in child processes
    (isolated: a failure or hang cannot take the main measurement with it),
    with the reduced-size oracle parity check first.  Rank 0 prints JSON."""
    import torch
    import torch.distributed as dist

    import paper_1511_04561_b200 as A
    from oracle import approx8_oracle as O

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idx = int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count()
    dev = torch.device("cuda", idx)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    spec = A.parse_spec(SPEC_LABEL)
    tr = A.SymmetricMemoryTransport()
    # parity: reduced AlexNet-shaped tensors, 2 calls, against the composed oracle
    small = [[np.random.default_rng(1000 + 16 * r + t).normal(0.0, SIGMA, n0).astype(np.float32)
              for t, (n0,) in enumerate(PARITY_SIZES)] for r in range(world)]
    want = (O.exchange_allgather(small, "dynamic-tree", "absmax", op="avg") if mode == "allgather"
            else O.exchange_two_round(small, "dynamic-tree", "absmax", op="avg"))
    pex_small = A.PeerExchange(spec, tr, mode=mode, check="sync")
    ok = True
    for _ in range(2):
        mine = [torch.from_numpy(g).to(dev) for g in small[rank]]
        pex_small(mine)
        ok &= all(m.cpu().numpy().tobytes() == w.astype(np.float32).tobytes() for m, w in zip(mine, want))
    grads = [torch.from_numpy(g).to(dev) for g in alexnet_grads(rank)]
    n = sum(g.numel() for g in grads)
    outs = [torch.empty_like(g) for g in grads]
    pex = A.PeerExchange(spec, tr, mode=mode, check="deferred")
    for _ in range(3):
        pex(grads, out=outs)
    pex.synchronize()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[idx])
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(steps):
        pex(grads, out=outs)
    a1.record()
    torch.cuda.synchronize()
    pex.synchronize()
    t = torch.tensor([a0.elapsed_time(a1) / steps, 0.0 if ok else 1.0], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t[0].item())
        print(json.dumps({"value": world * 4.0 * n / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                          "mode": mode, "parity_reduced_sizes": bool(t[1].item() == 0.0),
                          "how": "PeerExchange: encode into this rank's slab of a torch symmetric-memory buffer, "
                                 "device barrier, a8_decode_peers reads every rank's codes over NVLink"}), flush=True)
    dist.destroy_process_group()


# ---------------------------------------------------------------------------
# N = 1: the other BASELINE configs' codec numbers, measured in the same run


def codec_sweep(A, torch, dev, clk_sampler_cls):
    """Config 1 (2^20 round trip, 4 codebooks), config 4 at 2^28 and 2^30
    (dynamic-tree/absmax and mantissa/decade+1) and the per-block absmax codec
    at 2^30 (blocks of 4096 and 1024): encode / decode kernel time of one
    public-API call each (captured in a CUDA graph, replayed between CUDA
    events; L2 flushed before every replay by READING a 256 MB buffer, so the
    flush leaves clean lines and adds no write-back of its own to the timed
    region -- a written flush buffer left ~126 MB dirty in L2 that every
    measurement then wrote back, ~19 us), with its own clocks record.
    Synthetic N(0, 1) inputs generated on the device."""
    flush = torch.zeros(64 << 20, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    sink = torch.zeros((), dtype=torch.float32, device=dev)
    peak, _ = peaks()

    def time_graph(fn, reps):
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            fn()  # allocations happen here, outside the capture
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        ts = []
        for _ in range(reps):
            torch.sum(flush, 0, out=sink)  # read flush: evicts L2 (and writes back its dirty lines) before e0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts))

    def case(n, label, block=None):
        spec = A.parse_spec(label)
        cb = A.build_codebook(spec)
        x = torch.randn(n, device=dev)
        y = torch.empty_like(x)
        box = {}

        def enc():
            box["q"] = A.encode_buffer(x, cb, sync=False, block_size=block)

        def dec():
            A.decode_buffer(box["q"], cb, out=y)

        reps = 7 if n >= 1 << 28 else 15
        te = time_graph(enc, reps)
        box["q"]._finish()
        td = time_graph(dec, reps)
        r = {"n": n, "spec": label, "encode_ms": te, "decode_ms": td,
             "encode_GBps": 5.0 * n / (te * 1e-3) / 1e9, "decode_GBps": 5.0 * n / (td * 1e-3) / 1e9,
             "roundtrip_GBps": 10.0 * n / ((te + td) * 1e-3) / 1e9}
        r["roundtrip_frac"] = r["roundtrip_GBps"] / peak
        if block:
            r["block"] = block
        del x, y, box
        return r

    def premax_c4(n):
        """encode_buffer given the producer's max (one pass) vs computing it."""
        cb = A.build_codebook(A.parse_spec("dynamic-tree/absmax"))
        x = torch.randn(n, device=dev)
        m = A.scale_absmax_([x], 1.0)
        box = {}
        t2 = time_graph(lambda: box.__setitem__("q", A.encode_buffer(x, cb, sync=False)), 7)
        t1 = time_graph(lambda: box.__setitem__("q", A.encode_buffer(x, cb, sync=False, amax=m)), 7)
        box["q"]._finish()
        tm = time_graph(lambda: A.scale_absmax_([x], 1.0), 7)
        del x, box
        return {"n": n, "spec": "dynamic-tree/absmax", "encode_two_pass_ms": t2, "encode_premax_ms": t1,
                "max_pass_ms": tm, "encode_premax_GBps": 5.0 * n / (t1 * 1e-3) / 1e9,
                "encode_premax_frac": 5.0 * n / (t1 * 1e-3) / 1e9 / peak}

    def premax_c3():
        """Config-3 gradients through a producer pass (the data-parallel 1/2
        pre-scale) and the N=1 exchange: torch's multiply + the two-pass
        encode, against the fused producer + the one-pass encode."""
        spec = A.parse_spec("dynamic-tree/absmax")
        ts = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in ALEXNET]
        ex1, ex2 = A.GradientExchange(spec, check="none"), A.GradientExchange(spec, check="none")
        half = 0.5

        def two_pass():
            torch._foreach_mul_(ts, half)
            ex1(ts)

        def fused():
            ex2(ts, amax=A.scale_absmax_(ts, half))

        # the encode alone (one multi-tensor launch, as the exchange issues it)
        from paper_1511_04561_b200.exchange import CudaSegmentCodec, make_plan

        plan = make_plan(tuple(t.numel() for t in ts), 1)
        C, P = plan.flat, plan.allgather_block()
        slab = torch.zeros(P, dtype=torch.uint8, device=dev)
        cb, codec, idx = A.build_codebook(spec), CudaSegmentCodec(), list(range(plan.nseg))
        m = A.scale_absmax_(ts, 1.0)

        def enc(**kw):
            codec.encode(ts, plan.offs, idx, cb, slab, 0, C, C, C, 0, 1, C + 4 * plan.status_slot, **kw)

        n_el = sum(t.numel() for t in ts)
        te2, te1 = time_graph(enc, 15), time_graph(lambda: enc(amax=m), 15)
        r = {"encode_two_pass_ms": te2, "encode_premax_ms": te1,
             "encode_premax_frac": 5.0 * n_el / (te1 * 1e-3) / 1e9 / peak,
             "encode_two_pass_frac": 5.0 * n_el / (te2 * 1e-3) / 1e9 / peak}
        r.update({"tensors": len(ts), "elements": n_el,
             "torch_scale_then_exchange_ms": time_graph(two_pass, 15),
             "fused_scale_absmax_then_premax_exchange_ms": time_graph(fused, 15),
             "exchange_alone_ms": time_graph(lambda: ex1(ts), 15),
             "max_pass_then_premax_exchange_ms": time_graph(lambda: ex2(ts, amax=A.scale_absmax_(ts, 1.0)), 15)})
        del ts, slab
        return r

    def onebit_c3():
        """The 1-bit error-feedback exchange (GradientExchange("onebit"),
        mlp.py:313-321) over the config-3 gradients at N = 1: quantize
        (float64 residual per tensor) + the fused level decode, one step."""
        ts = [torch.randn(int(np.prod(s)), device=dev) * 1e-3 for s in ALEXNET]
        outs = [torch.empty_like(t) for t in ts]
        ex = A.GradientExchange("onebit", check="none")
        n_el = sum(t.numel() for t in ts)
        ex(ts, out=outs)  # residuals allocated
        torch.cuda.synchronize()
        try:
            ms, how = time_graph(lambda: ex(ts, out=outs), 15), "graph"
        except Exception:  # noqa: BLE001  (eager timing if the step cannot be captured)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(15):
                ex(ts, out=outs)
            e1.record()
            torch.cuda.synchronize()
            ms, how = e0.elapsed_time(e1) / 15, "eager"
        del ts, outs
        # bytes: quantize reads g + residual twice, writes residual + bits; decode writes out
        return {"elements": n_el, "step_ms": ms, "timing": how,
                "fp32_equiv_GBps": 4.0 * n_el / (ms * 1e-3) / 1e9,
                "hbm_GBps_at_32B_per_elem": 32.0 * n_el / (ms * 1e-3) / 1e9}

    out = {}
    with clk_sampler_cls(dev.index) as clk:
        out["c1"] = [case(1 << 20, lab) for lab in ("dynamic-tree/absmax", "linear/absmax", "static-tree/decade+1",
                                                    "mantissa/decade+1")]
        out["c4"] = [case(1 << k, lab) for k in (28, 30) for lab in ("dynamic-tree/absmax", "mantissa/decade+1")]
        out["blocked"] = [case(1 << k, "dynamic-tree/absmax", b) for k in (28, 30) for b in (4096, 1024)]
        out["premax"] = {"c4": [premax_c4(1 << k) for k in (28, 30)], "c3": premax_c3()}
        out["onebit_c3"] = onebit_c3()
    out["clocks"] = clk.summary()
    out["how"] = ("one public-API encode_buffer / decode_buffer call per case, CUDA-graph replayed between events, "
                  "median of 7-15, L2 flushed before each by reading 256 MB (clean lines: no flush write-back in the timed region); GB/s at 5 B/elem each way, round trip 10 B/elem; "
                  "frac against MEASURED_PEAKS hbm_gbs")
    del flush
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# the B200 arm


def run_b200(args, nranks, rank, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1511_04561_b200 as A

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    spec = A.parse_spec(SPEC_LABEL)
    host = alexnet_grads(rank)
    n = sum(g.size for g in host)
    pinned = [torch.from_numpy(g).pin_memory() for g in host]
    grads = [p.to(dev) for p in pinned]
    outs = [torch.empty_like(g) for g in grads]
    # one rank: the step is captured in a CUDA graph (one launch per step, no
    # host work between the kernels); N > 1 runs eagerly (NCCL in the step)
    graphed = nranks == 1 and not args.eager
    ex = A.GradientExchange(spec, mode=args.mode, op="avg", check="deferred", graph=graphed)

    def barrier():
        if nranks > 1:
            if dist.get_backend() == "nccl":
                dist.barrier(device_ids=[dev.index])
            else:
                dist.barrier()

    def max_over_ranks(v):
        if nranks == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # per-kernel event timing: a second exchange of the same step whose codec
    # calls are wrapped in CUDA events (in graph mode the event nodes are
    # captured into its graph).  The timed region runs `ex`, whose graph has
    # no event nodes -- they cost ~15 us per step (4 event records between
    # the kernels break the graph's kernel-to-kernel launch pipelining) --
    # and the kernel durations come from `steps` replays of the evented one.
    ex_t = A.GradientExchange(spec, mode=args.mode, op="avg", check="deferred", graph=graphed)
    codec = ex_t.codec
    ev_log = []

    class TimedCodec:
        """CUDA events on the launching stream around every codec call.  The
        events are `external` so that, in graph mode, they are captured into
        the graph and re-recorded by every replay."""

        def _timed(self, name, fn, *a, **k):
            e0 = torch.cuda.Event(enable_timing=True, external=graphed)
            e1 = torch.cuda.Event(enable_timing=True, external=graphed)
            e0.record()
            fn(*a, **k)
            e1.record()
            ev_log.append((name, e0, e1))

        def encode(self, *a, **k):
            self._timed("encode", codec.encode, *a, **k)

        def decode(self, *a, **k):
            self._timed("decode", codec.decode, *a, **k)

    ex_t.codec = TimedCodec()

    for _ in range(args.warmup):
        ex(grads, out=outs)
        ex_t(grads, out=outs)
    ex.synchronize()
    ex_t.synchronize()
    torch.cuda.synchronize()
    # graph mode: the events of the captured step (the codec calls of the
    # capture are the last ones logged; replays log nothing)
    captured = list(ev_log[-2:]) if graphed else []
    ev_log.clear()

    def soak(seconds):
        """Untimed steps around the timed region so the clock sampler (100 ms
        period) sees the GPU under this load before and after it."""
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(10):
                ex(grads, out=outs)
            torch.cuda.synchronize()

    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        soak(0.6)
        barrier()
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            ex(grads, out=outs)
        stop.record()
        torch.cuda.synchronize()
        barrier()
        # per-kernel durations, same step through the evented exchange:
        # graph mode, the captured events read after each of `steps` replays
        # (the replay that re-records them runs the same graph); eager mode,
        # the events logged by `steps` back-to-back calls
        kt: dict = {}
        ev_log.clear()
        if graphed:
            for _ in range(args.steps):
                ex_t(grads, out=outs)
                torch.cuda.synchronize()
                for name, e0, e1 in captured:
                    kt.setdefault(name, []).append(e0.elapsed_time(e1))
        else:
            for _ in range(args.steps):
                ex_t(grads, out=outs)
        ex_t.synchronize()
        torch.cuda.synchronize()
        soak(0.3)
    ms = start.elapsed_time(stop) / args.steps
    ms = max_over_ranks(ms)
    value = nranks * 4.0 * n / (ms * 1e-3) / 1e9
    for name, e0, e1 in ev_log:
        kt.setdefault(name, []).append(e0.elapsed_time(e1))
    kms = {k: float(np.mean(v)) * len(v) / args.steps for k, v in kt.items()}  # ms per step
    launches = {k: len(v) for k, v in kt.items()}
    nseg = len(ALEXNET)
    if args.mode == "allgather" or nranks == 1:
        alg = {"encode": 5.0 * n + 4 * nseg, "decode": (nranks + 4.0) * n + 4 * nranks * nseg}
    else:
        alg = {"encode": 5.0 * n + 5.0 * n / nranks, "decode": (nranks + 4.0) * n / nranks + 5.0 * n}
    dom = max(kms, key=lambda k: kms[k])
    per_launch_ms = float(np.mean(kt[dom]))
    per_launch_bytes = alg[dom] / (len(kt[dom]) / args.steps)
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        traffic = json.loads(tj.read_text()).get(f"{dom}_n{nranks}")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": per_launch_bytes,
                "traffic_note": ("encode: per-tensor absmax is two passes, so the inputs are read twice "
                                 f"({4.0 * n / 1e6:.0f} MB of re-read beyond the algorithmic 5 B/elem; L2 keeps "
                                 "little of it, DESIGN.md §3); traffic = ncu dram bytes of one launch "
                                 "(profiles/ncu_traffic.json, cold L2)") if dom == "encode" else None,
                "kernel_ms_per_step": kms,
                "codec_roundtrip_GBps": (alg["encode"] + alg["decode"]) / ((kms["encode"] + kms["decode"]) * 1e-3) / 1e9}

    # N > 1: parity of this exchange path on NCCL (reduced sizes vs the
    # oracle, and every rank holding the same C3 result), then the 32-bit
    # NCCL all-reduce of the same gradient (north-star comparison), with
    # NCCL_ALGO=Ring and with NCCL's default choice
    nccl = None
    parity = None
    peer = None
    if nranks > 1:
        ex.synchronize()
        agree, digest = outputs_agree(dist, outs, nranks)
        small_ok, blocks = parity_small(A, dist, args.mode, nranks, rank, dev)
        flags = torch.tensor([int(small_ok)], device=dev)
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        parity = {"ok": bool(agree and int(flags.item())), "ranks_agree_c3": agree, "c3_digest": digest,
                  "oracle_reduced_sizes": bool(int(flags.item())), "reduced_sizes": [n0 for (n0,) in PARITY_SIZES],
                  "how": "same GradientExchange path (mode, NCCL collectives, pipelined chunk blocks) on reduced "
                         "AlexNet-shaped tensors vs the composed oracle, bit-exact on every rank; C3 outputs "
                         "identical (sha256) on every rank"}
        legs = {}
        if dist.get_backend() == "nccl":
            for algo in ("Ring", "default"):
                legs[algo] = nccl_leg(dist, algo, n, args.steps, rank, nranks, local_rank)
        else:  # A8_BENCH_BACKEND=gloo plumbing runs (ranks sharing one GPU): NCCL cannot run there
            legs = {"skipped": f"backend {dist.get_backend()}"}
        nccl = {"legs": legs}
        if dist.get_backend() == "nccl" and os.environ.get("A8_BENCH_PEER", "1") == "1":
            peer = nccl_leg(dist, "default", n, args.steps, rank, nranks, local_rank,
                            child_args=["--peer-leg", args.mode])
        else:
            peer = {"skipped": f"backend {dist.get_backend()}"}
        for algo, leg in legs.items():
            if isinstance(leg, dict) and "value" in leg:
                leg["speedup_8bit"] = value / leg["value"]

    # NVLink roofline of the exchange: bytes each rank must
    # receive over NVLink per step / the measured peer-copy bandwidth
    # (770 GB/s per direction, B200_PROFILING.md), against the step time
    nvlink = None
    if nranks > 1:
        if args.mode == "allgather":
            ingress = (nranks - 1) * (n + 4 * len(ALEXNET))
        else:  # two_round: an all-to-all of 8-bit shards, then an all-gather of them
            ingress = 2 * (nranks - 1) * n / nranks
        bound_ms = ingress / 770e9 * 1e3
        nvlink = {"ingress_bytes_per_rank": ingress, "peer_GBps": 770.0, "bound_ms": bound_ms,
                  "frac": bound_ms / ms, "fp32_ring_allreduce_ingress_bytes": 2 * (nranks - 1) / nranks * 4.0 * n}

    # e2e: host buffers through the public API, copies inside the timed region.
    # Every step copies its gradients host->device (pinned), exchanges them
    # and copies the averaged result device->host.  Steps are software
    # pipelined over two device buffers on three streams, so the H2D of
    # step k+1 and the D2H of step k use both PCIe directions at once.
    NB = 2  # device buffers in flight (3 measured no better: the copies share PCIe)
    host_out = [[torch.empty_like(p).pin_memory() for p in pinned] for _ in range(NB)]
    dev_in = [[torch.empty_like(g) for g in grads] for _ in range(NB)]
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(NB)]
    ev_done = [torch.cuda.Event() for _ in range(NB)]
    ev_out = [torch.cuda.Event() for _ in range(NB)]
    for b in range(NB):  # buffers start free
        ev_done[b].record(comp)
        ev_out[b].record(comp)

    def e2e_step(i):
        b = i % NB
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(ev_out[b])  # the previous D2H from this buffer has finished
            for d, p in zip(dev_in[b], pinned):
                d.copy_(p, non_blocking=True)
            ev_in[b].record(s_h2d)
        comp.wait_event(ev_in[b])
        ex(dev_in[b])
        ev_done[b].record(comp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_done[b])
            for h, d in zip(host_out[b], dev_in[b]):
                h.copy_(d, non_blocking=True)
            ev_out[b].record(s_d2h)

    for i in range(max(NB, args.warmup)):
        e2e_step(i)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    for i in range(args.steps):
        e2e_step(i)
    for b in range(NB):
        comp.wait_event(ev_out[b])
    e1.record(comp)
    torch.cuda.synchronize()
    barrier()
    ex.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    # the PCIe bound of that step: the same bytes copied H2D and D2H
    # concurrently (pinned), no compute
    a_in, a_out = torch.empty(n, device=dev), torch.empty(n, device=dev)
    h_in, h_out = torch.empty(n).pin_memory(), torch.empty(n).pin_memory()
    pcie = []
    for _ in range(3):
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(comp)
        s_h2d.wait_event(p0)
        s_d2h.wait_event(p0)
        with torch.cuda.stream(s_h2d):
            a_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s_d2h):
            h_out.copy_(a_out, non_blocking=True)
        comp.wait_stream(s_h2d)
        comp.wait_stream(s_d2h)
        p1.record(comp)
        torch.cuda.synchronize()
        pcie.append(p0.elapsed_time(p1))
    pcie_ms = float(np.median(pcie))
    del a_in, a_out, h_in, h_out
    e2e = {"value": nranks * 4.0 * n / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n, "ms_per_step": e2e_ms,
           "pcie_bound_ms": pcie_ms, "frac_of_pcie_bound": pcie_ms / e2e_ms,
           "how": f"pinned H2D + exchange + D2H every step, pipelined over {NB} buffers / 3 streams; "
                  "pcie_bound_ms = the same H2D and D2H bytes copied concurrently without compute"}

    cpu = None
    if rank == 0 and nranks == 1 and not args.no_cpu:
        # the reference's CPU implementation on this very workload (all 16
        # tensors, one full step, all host threads), plus one core
        rt, kind = reference_codec()
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        cpu_reference_step([host], 1, threads, rt)
        dt = time.perf_counter() - t0
        cpu = {"value": 4.0 * n / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
               "sample": f"one full step of this workload ({n} elements, 16 tensors over {threads} threads), "
                         + ("unmodified approx8 roundtrip (baseline/_ref)" if kind == "reference"
                            else "oracle port of approx8.codecs roundtrip"),
               "single_core": {"value": single_core_rate(rt), "unit": "GB/s", "cores": 1,
                               "sample": "one 2^22-element tensor, one round trip"}}

    sweep = None
    if rank == 0 and nranks == 1 and not args.no_sweep:
        sweep = codec_sweep(A, torch, dev, ClockSampler)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": nranks, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {**workload_config(args, nranks), "cuda_graph": graphed},
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clk.summary(), "gpu_launches": int(sum(launches.values())),
            "gpu_launches_per_step": {k: v / args.steps for k, v in launches.items()},
            "nccl_fp32_allreduce": nccl,
            "nvlink_roofline": nvlink,
            "parity": parity,
            "peer_exchange": peer,
            "codec_sweep": sweep,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "allgather", "two_round"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-1/4/per-block codec sub-measurements")
    ap.add_argument("--nccl-leg", type=int, default=0, help=argparse.SUPPRESS)  # child of nccl_leg()
    ap.add_argument("--peer-leg", default="", help=argparse.SUPPRESS)  # child: PeerExchange timing
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the N=1 step")
    args = ap.parse_args()
    if args.nccl_leg:
        nccl_leg_child(args.nccl_leg, args.steps)
        return
    if args.peer_leg:
        peer_leg_child(args.peer_leg, args.steps)
        return
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.mode == "auto":  # ingress (N-1)n vs 2(N-1)/N n: two_round wins from N = 4
        args.mode = "allgather" if max(world, args.gpus) <= 2 else "two_round"
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, max(world, args.gpus), rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        # A8_BENCH_BACKEND=gloo: plumbing check of the N > 1 path with every
        # rank on one GPU (ranks wrap around the visible devices); numbers
        # from such a run are not measurements
        backend = os.environ.get("A8_BENCH_BACKEND", "nccl")
        idx = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(idx)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", idx))
        else:
            dist.init_process_group(backend)
    try:
        run_b200(args, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
