"""bench.py's multi-rank logic on CPU (gloo, world size 2): one C4-style
batch sharded by row_blocks, each rank's output checked against per-image
reference digests and the per-iteration stat sums reduced over the ranks --
the parity gate that decides whether the bench prints a value.  The oracle
stands in for the GPU output here (tests/ may use it)."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(n):
    return [O.inject_sp_noise(O.synth_image(45, 29, i), bench.c4_density(i), 0.5, i) for i in range(n)]


def _golden(n, k=5):
    outs = [O.denoise(x, k=k) for x in _batch(n)]
    sums = np.zeros((k, 2), np.int64)
    for _, st in outs:
        for j, fr in enumerate(st):
            sums[j] += fr
    return {"n": n, "final_per_image": [hashlib.sha256(o.tobytes()).hexdigest()[:16] for o, _ in outs],
            "stats_sum": sums.tolist()}


def _reduce(x, op):
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}[op])
    return float(t.item())


def _worker(rank, world, port, n, corrupt):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _golden(n)
        i0, i1 = bench.shard(n, world, rank)
        imgs = _batch(n)[i0:i1]
        out = np.stack([O.denoise(x)[0] for x in imgs])
        ctr = np.zeros((i1 - i0, 5, 2), np.int64)
        for i, x in enumerate(imgs):
            for j, fr in enumerate(O.denoise(x)[1]):
                ctr[i, j] = fr
        if corrupt and rank == world - 1:
            out[0, 5, 5] ^= 1
        res = bench.parity_batch_shard(out, ctr, i0, g, _reduce)
        assert res["checked"] and res["ok"] == (not corrupt), res
        assert res["images_differing"] == (1 if corrupt else 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_sharded_batch_parity_gate_over_gloo(corrupt):
    mp.spawn(_worker, args=(2, _free_port(), 13, corrupt), nprocs=2, join=True)


def test_shards_and_truncation():
    assert [bench.shard(4096, 8, r) for r in (0, 7)] == [(0, 512), (3584, 4096)]
    assert sum(hi - lo for lo, hi in (bench.shard(4096, 3, r) for r in range(3))) == 4096
    assert bench.truncated([[5, 3], [2, 0], [0, 0]]) == [[5, 3], [2, 0]]
