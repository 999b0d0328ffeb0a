"""Multi-GPU parity of the compressed exchange over NCCL (one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/nccl_parity.py

Every rank runs, on its own GPU with the NCCL backend:
  * allgather and two_round (op avg and sum) at reduced AlexNet-shaped sizes,
    pipelined chunk blocks forced (chunk_elems 64K), against the composed
    oracle (oracle/approx8_oracle.py) bit for bit;
  * the paper's local-fp32 variant against its oracle;
  * the full config-3 AlexNet shapes (61,100,840 elements per rank,
    bench.py's gradients) in both modes: outputs identical on every rank, and
    for allgather a sampled oracle check (the sampled elements' per-tensor
    round trips, gathered and averaged in rank order);
  * the DDP comm hook (a8_comm_hook) on a real DistributedDataParallel model.
Prints one JSON line per rank; exit status 0 iff every check passed.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1511_04561_b200 as A  # noqa: E402
from oracle import approx8_oracle as O  # noqa: E402

import bench  # noqa: E402  (the config-3 gradients)

SPEC = A.DataTypeSpec("dynamic-tree", "absmax")


def small(r, seed=0):
    out = []
    for t, (n,) in enumerate(bench.PARITY_SIZES):
        rng = np.random.default_rng(seed + 1000 + 16 * r + t)
        out.append(rng.normal(0.0, 1e-3, n).astype(np.float32))
    return out


def check_small(world, rank, dev):
    res = {}
    per = [small(r) for r in range(world)]
    for mode in ("allgather", "two_round"):
        for op in ("avg", "sum"):
            want = (O.exchange_allgather(per, "dynamic-tree", "absmax", op=op) if mode == "allgather"
                    else O.exchange_two_round(per, "dynamic-tree", "absmax", op=op))
            ex = A.GradientExchange(SPEC, mode=mode, op=op, check="sync", chunk_elems=1 << 16)
            mine = [torch.from_numpy(g).to(dev) for g in per[rank]]
            ex(mine)
            res[f"{mode}_{op}"] = all(m.cpu().numpy().tobytes() == w.astype(np.float32).tobytes()
                                      for m, w in zip(mine, want))
    want = O.exchange_allgather_local(per, rank, "dynamic-tree", "absmax")
    ex = A.GradientExchange(SPEC, check="sync", local_fp32=True, chunk_elems=1 << 16)
    mine = [torch.from_numpy(g).to(dev) for g in per[rank]]
    ex(mine)
    res["local_fp32"] = all(m.cpu().numpy().tobytes() == w.astype(np.float32).tobytes() for m, w in zip(mine, want))
    # non-finite input on one rank raises on every rank
    bad = [torch.from_numpy(g).to(dev) for g in per[rank]]
    if rank == world - 1:
        bad[3][0] = float("nan")
    try:
        A.GradientExchange(SPEC, check="sync")(bad)
        res["nonfinite_raises"] = False
    except A.InputError:
        res["nonfinite_raises"] = True
    return res


def check_peer(world, rank, dev):
    """PeerExchange over torch symmetric memory (the decode reads the peers'
    slabs over NVLink) against the same oracles, 2 calls per mode."""
    res = {}
    tr = A.SymmetricMemoryTransport()
    for mode in ("allgather", "two_round"):
        ex = A.PeerExchange(SPEC, tr, mode=mode, op="avg", check="sync")
        ok = True
        for step in range(2):
            per = [small(r, seed=10 * step) for r in range(world)]
            want = (O.exchange_allgather(per, "dynamic-tree", "absmax", op="avg") if mode == "allgather"
                    else O.exchange_two_round(per, "dynamic-tree", "absmax", op="avg"))
            mine = [torch.from_numpy(g).to(dev) for g in per[rank]]
            ex(mine)
            ok &= all(m.cpu().numpy().tobytes() == w.astype(np.float32).tobytes() for m, w in zip(mine, want))
        res[f"peer_{mode}"] = bool(ok)
    return res


def check_c3(world, rank, dev):
    res = {}
    host = bench.alexnet_grads(rank)
    rng = np.random.default_rng(7)
    samples = [np.unique(np.concatenate([[0, g.size - 1], rng.integers(0, g.size, 2000)])) for g in host]
    # this rank's round trip of the sampled elements, with the full-tensor scale (codecs.py:232-288)
    table = O.book("dynamic-tree").table
    mine = []
    for g, idx in zip(host, samples):
        flat = g.reshape(-1)
        s = O.scale_of(flat, "absmax")
        c = O.encode_by_thresholds(flat[idx], "dynamic-tree", s)
        mine.append((table[c] * np.float32(s)).astype(np.float32))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    for mode in ("allgather", "two_round"):
        ts = [torch.from_numpy(g).to(dev) for g in host]
        A.GradientExchange(SPEC, mode=mode, op="avg", check="sync")(ts)
        outs = [t.reshape(-1).cpu().numpy() for t in ts]
        import hashlib

        h = hashlib.sha256(b"".join(o.tobytes() for o in outs)).hexdigest()
        digests = [None] * world
        dist.all_gather_object(digests, h)
        res[f"c3_{mode}_ranks_agree"] = len(set(digests)) == 1
        if mode == "allgather":
            ok = True
            for t, idx in enumerate(samples):
                acc = gathered[0][t].copy()
                for r in range(1, world):
                    acc = (acc + gathered[r][t]).astype(np.float32)
                acc = (acc / np.float32(world)).astype(np.float32)
                ok &= outs[t][idx].tobytes() == acc.tobytes()
            res["c3_allgather_sampled_oracle"] = bool(ok)
    return res


def check_ddp(world, rank, dev):
    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(20, 30), torch.nn.ReLU(), torch.nn.Linear(30, 5)).to(dev)
    ref = [p.detach().clone() for p in model.parameters()]
    ddp = torch.nn.parallel.DistributedDataParallel(model, device_ids=[dev.index])
    ddp.register_comm_hook(A.DDPHookState(SPEC, check="sync"), A.a8_comm_hook)

    def inputs(r):
        g = torch.Generator().manual_seed(100 + r)
        return torch.randn(8, 20, generator=g), torch.randn(8, 5, generator=g)

    x, y = inputs(rank)
    torch.nn.functional.mse_loss(ddp(x.to(dev)), y.to(dev)).backward()
    per_rank = []
    for r in range(world):
        m = torch.nn.Sequential(torch.nn.Linear(20, 30), torch.nn.ReLU(), torch.nn.Linear(30, 5)).to(dev)
        with torch.no_grad():
            for p, q in zip(m.parameters(), ref):
                p.copy_(q)
        xr, yr = inputs(r)
        torch.nn.functional.mse_loss(m(xr.to(dev)), yr.to(dev)).backward()
        per_rank.append([p.grad.cpu().numpy().copy() for p in m.parameters()])
    ok = True
    for i, p in enumerate(model.parameters()):
        want = O.exchange_allgather([[per_rank[r][i]] for r in range(world)], "dynamic-tree", "absmax", op="avg")[0]
        ok &= bool(np.array_equal(p.grad.cpu().numpy(), want))
    return {"ddp_hook": ok}


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    idx = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(idx)
    dev = torch.device("cuda", idx)
    dist.init_process_group("nccl", device_id=dev)
    try:
        res = {"rank": rank, "world": world, "backend": dist.get_backend()}
        res.update(check_small(world, rank, dev))
        res.update(check_ddp(world, rank, dev))
        if os.environ.get("A8_PARITY_PEER", "1") == "1":
            try:
                res.update(check_peer(world, rank, dev))
            except Exception as exc:  # noqa: BLE001  (report, do not hide: ok becomes False)
                res["peer_error"] = repr(exc)[:300]
                res["peer_ok"] = False
        if os.environ.get("A8_PARITY_C3", "1") == "1":
            res.update(check_c3(world, rank, dev))
        res["ok"] = all(v for k, v in res.items() if isinstance(v, bool))
        print(json.dumps(res), flush=True)
    finally:
        dist.destroy_process_group()
    sys.exit(0 if res["ok"] else 1)


if __name__ == "__main__":
    main()
