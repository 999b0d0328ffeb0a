"""Benchmark of the 8-bit approximation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--mode allgather|two_round] [--workload c3|c1|sweep]

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
+ synchronize around the K timed steps, max over ranks.
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
# reference arm / CPU baseline: the oracle port of approx8.codecs on host cores


def cpu_reference_step(sample, nranks: int, threads: int):
    """One step of the reference algorithm on a bounded sample: every rank's
    tensors are encoded+decoded (codecs.py:244-288) and accumulated in rank
    order (the composed exchange); tensors are spread over the threads."""
    from oracle import approx8_oracle as O

    def work(i):
        acc = None
        for r in range(nranks):
            d = O.roundtrip(sample[r][i], "dynamic-tree", "absmax")
            acc = d if acc is None else acc + d
        return acc / np.float32(nranks) if nranks > 1 else acc

    with cf.ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(work, range(len(sample[0]))))


def cpu_sample(nranks: int, threads: int, elems: int):
    """Bounded sample of the config-3 workload: `threads` independent
    tensors of `elems/threads` elements per rank, N(0, sigma)."""
    per = max(1, elems // threads)
    out = []
    for r in range(nranks):
        rng = np.random.default_rng(1000 + 16 * r)
        out.append([rng.normal(0.0, SIGMA, per).astype(np.float32) for _ in range(threads)])
    return out, per * threads


def run_reference(args, nranks, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample, n = cpu_sample(nranks, threads, args.cpu_elems)
    for _ in range(args.warmup):
        cpu_reference_step(sample, nranks, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_reference_step(sample, nranks, threads)
    dt = (time.perf_counter() - t0) / args.steps
    value = nranks * 4.0 * n / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": nranks,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args, nranks),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{nranks} rank(s) x {threads} tensors x {n // threads} elems "
                                   f"N(0,{SIGMA}) per step, reference algorithm (oracle port of "
                                   f"approx8.codecs encode/decode + rank-ordered average)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, nranks):
    n = sum(int(np.prod(s)) for s in ALEXNET)
    return {"workload": "C3 AlexNet-sized synthetic gradient exchange", "elements_per_rank": n,
            "tensors": len(ALEXNET), "spec": SPEC_LABEL, "scale": "per-tensor absmax",
            "mode": args.mode if nranks > 1 else "roundtrip (N=1)", "op": "avg",
            "parallelism": f"dp{nranks}", "l2": "inputs 244 MB/rank > 126 MB L2, no flush"}


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

    # per-kernel event timing: wrap the codec calls of this exchange
    codec = ex.codec
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

    ex.codec = TimedCodec()

    for _ in range(args.warmup):
        ex(grads, out=outs)
    ex.synchronize()
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
        ex.codec = codec
        soak(0.6)
        ex.codec = TimedCodec()
        ev_log.clear()
        barrier()
        torch.cuda.synchronize()
        start.record()
        for _ in range(args.steps):
            ex(grads, out=outs)
        stop.record()
        torch.cuda.synchronize()
        barrier()
        ex.codec = codec
        soak(0.3)
    ms = start.elapsed_time(stop) / args.steps
    ms = max_over_ranks(ms)
    value = nranks * 4.0 * n / (ms * 1e-3) / 1e9

    # per-kernel durations: eager mode, the events logged inside the timed
    # region; graph mode, the captured events read after each of `steps`
    # further replays (the replay that re-records them runs the same graph)
    kt: dict = {}
    if graphed:
        for _ in range(args.steps):
            ex(grads, out=outs)
            torch.cuda.synchronize()
            for name, e0, e1 in captured:
                kt.setdefault(name, []).append(e0.elapsed_time(e1))
        ex.synchronize()
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
                "kernel_ms_per_step": kms,
                "codec_roundtrip_GBps": (alg["encode"] + alg["decode"]) / ((kms["encode"] + kms["decode"]) * 1e-3) / 1e9}

    # north-star comparison at N > 1: a 32-bit NCCL all-reduce of the same
    # gradient bucket (one flat fp32 buffer), fp32-equivalent GB/s
    nccl = None
    if nranks > 1:
        flat = torch.cat([g.reshape(-1) for g in grads])
        for _ in range(3):
            dist.all_reduce(flat)
        torch.cuda.synchronize()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.steps):
            dist.all_reduce(flat)
        a1.record()
        torch.cuda.synchronize()
        nms = max_over_ranks(a0.elapsed_time(a1) / args.steps)
        nccl = {"value": nranks * 4.0 * n / (nms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": nms,
                "algo": os.environ.get("NCCL_ALGO", "default"), "speedup_8bit": value / (nranks * 4.0 * n / (nms * 1e-3) / 1e9)}
        del flat

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
    ex.codec = codec
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
        threads = os.cpu_count() or 1
        sample, sn = cpu_sample(1, threads, args.cpu_elems)
        cpu_reference_step(sample, 1, threads)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            cpu_reference_step(sample, 1, threads)
            reps += 1
        dt = (time.perf_counter() - t0) / reps
        cpu = {"value": 4.0 * sn / dt / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"{threads} tensors x {sn // threads} elems N(0,{SIGMA}), {reps} reps, "
                         f"reference algorithm (oracle port of approx8.codecs round trip)"}

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
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "allgather", "two_round"])
    ap.add_argument("--cpu-elems", type=int, default=1 << 23)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eager", action="store_true", help="no CUDA graph for the N=1 step")
    args = ap.parse_args()
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
