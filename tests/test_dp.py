"""Data-parallel host logic on CPU: microbatch assignment and the bucketed adapter-gradient
all-reduce over a world_size-2 gloo group (the NCCL path on the B200 box is identical)."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_00206_b200 import dp


def test_assign_microbatches_balances_and_covers():
    counts = [8192, 8000, 7800, 4096, 4096, 2048, 1024, 512, 8192, 6000, 300, 64]
    for world in (1, 2, 4, 8):
        a = dp.assign_microbatches(counts, world)
        flat = sorted(i for r in a for i in r)
        assert flat == list(range(len(counts)))
        loads = dp.rank_loads(counts, a)
        # LPT bound: max load <= mean + largest item
        assert max(loads) <= sum(counts) / world + max(counts)
        assert a == dp.assign_microbatches(counts, world)  # deterministic
    assert dp.imbalance([10, 10]) == 0.0
    assert dp.imbalance([10, 5]) == pytest.approx(1 - 7.5 / 10)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(rank)
        params = [torch.nn.Parameter(torch.zeros(16, 40)), torch.nn.Parameter(torch.zeros(72, 16)),
                  torch.nn.Parameter(torch.zeros(8, 8))]
        for i, p in enumerate(params):
            p.grad = torch.full_like(p, float(rank + 1) * (i + 1))
        params[2].grad = None  # a parameter without a gradient this step contributes zeros
        red = dp.AdapterGradReducer(params, bucket_bytes=3000)  # forces several buckets
        assert len(red.buckets) >= 2
        red.reduce()
        tot = sum(r + 1 for r in range(world))
        ok = all(torch.allclose(p.grad, torch.full_like(p, tot * (i + 1.0))) for i, p in enumerate(params[:2]))
        ok = ok and torch.count_nonzero(params[2].grad) == 0
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_adapter_grad_allreduce_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def _worker_overlap(rank: int, world: int, port: int, q):
    """attach/arm: buckets launch from post-accumulate-grad hooks during the last backward."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.manual_seed(0)
        lins = torch.nn.ModuleList(torch.nn.Linear(24, 24, bias=False) for _ in range(4))
        params = list(lins.parameters())
        red = dp.AdapterGradReducer(params, bucket_bytes=24 * 24 * 4 * 2).attach()  # 2 params per bucket
        x = torch.full((3, 24), float(rank + 1))
        launched_during_backward = []
        orig = red._launch_bucket

        def spy(b):
            launched_during_backward.append(b)
            orig(b)

        red._launch_bucket = spy
        for i in range(2):  # gradient accumulation: only the last backward is armed
            h = x
            for j, lin in enumerate(lins):
                # rank 1 skips layer 1 in its last microbatch (an adapter absent from it):
                # its bucket never completes there, yet collectives must stay matched
                if i == 1 and rank == 1 and j == 1:
                    continue
                h = lin(h)
            if i == 1:
                red.arm()
            h.sum().backward()
            if i == 0:
                ok0 = not launched_during_backward
        during = list(launched_during_backward)
        red.wait()
        # reference: local grads of both microbatches, summed over ranks
        ref = [torch.zeros_like(p) for p in params]
        for r in range(world):
            xr = torch.full((3, 24), float(r + 1))
            for i in range(2):
                ps = [p.detach().clone().requires_grad_(True) for p in params]
                h = xr
                for j, pw in enumerate(ps):
                    if i == 1 and r == 1 and j == 1:
                        continue
                    h = h @ pw.t()
                h.sum().backward()
                for acc, pw in zip(ref, ps):
                    if pw.grad is not None:
                        acc += pw.grad
        nb = len(red.buckets)
        ok = ok0 and launched_during_backward == list(range(nb))  # every bucket once, in order, on each rank
        ok = ok and (len(during) == nb if rank == 0 else 0 < len(during) < nb)  # hooks launched them (rank 1: up to the gap)
        ok = ok and all(torch.allclose(p.grad, g, rtol=1e-5) for p, g in zip(params, ref))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_adapter_grad_allreduce_overlapped_with_backward_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_overlap, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_c5_imbalance_matches_reference_simulate_dp():
    """The C5 bench leg's DP balance, restated by dp.imbalance over the LPT-assigned rank
    loads, equals lorasched's own simulate_dp on the same rank streams (linear time model;
    fixture generated from the reference by tests/golden/make_dp_golden.py)."""
    import json
    import os

    import bench
    from paper_2510_00206_b200 import dp as dp_

    with open(os.path.join(os.path.dirname(__file__), "golden", "c5_simulate_dp.json")) as f:
        gold = json.load(f)
    for world, ent in gold["worlds"].items():
        _, chosen, assign = bench.c5_microbatches(int(world), gold["microbatches_per_rank"])
        assert assign == ent["assignment"]
        loads = dp_.rank_loads([mb.rows for mb in chosen], assign)
        assert abs(dp_.imbalance(loads) - ent["linear"]["imbalance"]) < 1e-12
        # per-step max over ranks (simulate_dp's step cost) in rows, linear model: 1e-6 s/row x 3
        steps = [max(s[i] for s in ent["streams"]) for i in range(len(ent["streams"][0]))]
        assert abs(sum(steps) * 3e-6 - ent["linear"]["total_time_s"]) < 1e-9
