"""Multi-rank sharding logic on CPU (gloo, world sizes 2-4).

The row-band pipeline of paper_1306_5390_b200/dist.py -- row_blocks bands,
beta*Tmax halos, one P2P halo exchange per temporally blocked launch, one
all_reduce of the counters -- is driven with the oracle as the band stepper
(tests/ may use the oracle); the gathered result must equal the full-image
reference run bit for bit, stats included.  The GPU runs the same schedule
with the fused kernel as the stepper (bench.py --workload c5)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1306_5390_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_stepper(H, alpha, beta, thr, border, counters):
    def step(src, dst, plan, it0, iters):
        cur = src.numpy().copy()
        nxt = cur.copy()
        for i in range(iters):
            ext = beta * (iters - 1 - i)
            y_lo, y_hi = max(0, plan.lo - ext), min(H, plan.hi + ext)
            f, r = O.band_pass(cur, nxt, plan.blo, H, y_lo, y_hi, plan.lo, plan.hi, alpha, beta, thr, border)
            counters[it0 + i] += (f, r)
            cur, nxt = nxt, cur
        d = dst.numpy()
        d[plan.local(plan.lo):plan.local(plan.hi)] = cur[plan.local(plan.lo):plan.local(plan.hi)]
    return step


def _bands_worker(rank, world, port, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, density, seed, alpha, beta, k, thr, border, tmax = case
        img = O.inject_sp_noise(O.synth_image(W, H, seed), density, 0.5, seed + 1)
        plan = D.BandPlan(H, W, world, rank, beta * tmax)
        src = torch.from_numpy(np.ascontiguousarray(img[plan.blo:plan.bhi]))
        ta, tb = torch.zeros_like(src), torch.zeros_like(src)
        counters = np.zeros((k, 2), np.int64)
        out = D.denoise_band(src, ta, tb, plan, k, tmax, oracle_stepper(H, alpha, beta, thr, border, counters))
        ctr = D.reduce_counters(torch.from_numpy(counters))
        owned = out[plan.local(plan.lo):plan.local(plan.hi)].numpy().copy()
        parts = [None] * world
        dist.all_gather_object(parts, owned)
        full = np.concatenate(parts)
        ref, ref_stats = O.denoise(img, alpha, beta, k, thr, border)
        assert np.array_equal(full, ref), f"rank {rank}: image mismatch"
        assert D.truncate_stats(ctr) == ref_stats, (D.truncate_stats(ctr), ref_stats)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (97, 64, 0.3, 1, 20, 1, 5, 3, 0, 5)),
    (2, (64, 50, 0.5, 2, 20, 2, 5, 3, 1, 2)),
    (3, (81, 45, 0.2, 3, 30, 1, 7, 3, 0, 3)),
    (4, (40, 48, 0.6, 4, 20, 1, 5, 2, 1, 2)),
    # T = 1 launches (the C5 bench plan): a 1-row halo exchange after every
    # launch but the last
    (3, (70, 60, 0.3, 5, 20, 1, 5, 3, 0, 1)),
])
def test_row_bands_over_gloo_equal_full_image(world, case):
    mp.spawn(_bands_worker, args=(world, _free_port(), case), nprocs=world, join=True)


def _batch_worker(rank, world, port, n):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = D.shard(n, world, rank)
        mine = {}
        for i in range(lo, hi):
            img = O.inject_sp_noise(O.synth_image(33, 21, i), 0.1 + 0.6 * (i % 61) / 60, 0.5, i)
            mine[i] = O.denoise(img)[1]
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        merged = {}
        for p in parts:
            assert not (set(p) & set(merged)), "an image was processed twice"
            merged.update(p)
        assert sorted(merged) == list(range(n))
    finally:
        dist.destroy_process_group()


def test_batch_shards_cover_every_image_once():
    mp.spawn(_batch_worker, args=(3, _free_port(), 10), nprocs=3, join=True)


def test_band_plan_and_chunks():
    assert D.chunk_plan(5, 5) == [5] and D.chunk_plan(5, 4) == [3, 2] and D.chunk_plan(7, 1) == [1] * 7
    assert sum(D.chunk_plan(13, 4)) == 13
    plans = [D.BandPlan(100, 10, 4, r, 3) for r in range(4)]
    assert [(p.lo, p.hi) for p in plans] == [(0, 25), (25, 50), (50, 75), (75, 100)]
    assert (plans[0].blo, plans[0].bhi) == (0, 28) and (plans[3].blo, plans[3].bhi) == (72, 100)
    with pytest.raises(ValueError):
        D.BandPlan(10, 10, 4, 0, 3)  # bands thinner than the halo
    assert [D.shard(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
