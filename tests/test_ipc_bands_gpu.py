"""The multi-process row-band path with the halo exchange fused into the
launches (dist.IpcHaloPeers + dist.denoise_band_fused): G processes, each
owning one band, map their neighbours' ping-pong buffers with CUDA IPC and
the kernel epilogues store the neighbour-halo rows into them.  On one GPU
the G processes share the device (their kernels never wait on each other:
the launches are ordered by a host barrier), so the IPC mapping, the mirror
geometry and the launch ordering run exactly as on an NVSwitch node; the
result must equal the full-image oracle (denoise.hpp:292-311).  gloo carries
the handle exchange and the barriers."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [(2, 700, 260, 1, 12), (3, 600, 300, 1, 9), (2, 520, 200, 2, 9), (4, 400, 240, 2, 7)]


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1306_5390_b200 import dist as D
    from paper_1306_5390_b200._lib import PhgParams, lib

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _, W, H, beta, k = case
        torch.cuda.set_device(0)
        img = O.inject_sp_noise(O.synth_image(W, H, W + beta), 0.35, 0.5, 3)
        tmax = lib().phg_max_fused_iterations(beta)
        plan = D.BandPlan(H, W, world, rank, beta * tmax)
        pitch = (W + 15) // 16 * 16
        src = torch.zeros((plan.rows, pitch), dtype=torch.uint8, device="cuda")
        src[:, :W] = torch.from_numpy(img[plan.blo:plan.bhi]).cuda()
        bufs = [torch.zeros_like(src) for _ in range(2)]
        counters = torch.zeros((k, 2), dtype=torch.int64, device="cuda")
        peers = D.IpcHaloPeers(plan, bufs)
        step = D.cuda_band_stepper(PhgParams(20, beta, k, 3, 0), counters, W, H)
        out = D.denoise_band_fused(src, bufs, plan, k, tmax, step, peers)
        torch.cuda.synchronize()
        dist.barrier()  # nobody closes a mapping a neighbour may still write through
        peers.close()
        rows = out[plan.local(plan.lo):plan.local(plan.hi), :W].cpu().numpy()
        q.put((rank, rows, counters.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", CASES)
def test_ipc_fused_halo_bands_equal_full_image(case):
    from oracle import oracle as O
    from paper_1306_5390_b200 import dist as D

    world, W, H, beta, k = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    out = np.concatenate([r[1] for r in res])
    counters = sum(r[2] for r in res)
    img = O.inject_sp_noise(O.synth_image(W, H, W + beta), 0.35, 0.5, 3)
    ref, ref_stats = O.denoise(img, 20, beta, k, 3, 0)
    assert np.array_equal(out, ref)
    assert D.truncate_stats(torch.from_numpy(counters)) == ref_stats
