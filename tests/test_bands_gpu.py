"""The multi-GPU row-band schedule (paper_1306_5390_b200/dist.py) with the real
fused-kernel stepper, emulated as G bands on ONE device: the halo exchange is
a device copy between the band buffers instead of NCCL send/recv (the
gloo tests cover the torch.distributed plumbing)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_1306_5390_b200 import dist as D
from paper_1306_5390_b200._lib import PhgParams, lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,W,H,beta,k,border,tmax", [
    (2, 481, 321, 1, 5, 0, 0), (3, 700, 257, 2, 5, 1, 0), (4, 1000, 200, 1, 7, 0, 0), (8, 520, 400, 1, 5, 1, 0),
    # T = 1 launches: the single-buffer DIRECT form on wide regions (owned
    # rows of a band stored straight to HBM), the two-buffer form when narrow
    (3, 1500, 300, 1, 5, 0, 1), (2, 1100, 200, 2, 4, 0, 1), (2, 481, 321, 1, 3, 0, 1)])
def test_bands_on_one_device_equal_full_image(G, W, H, beta, k, border, tmax):
    lib().phg_set_device(0)
    img = O.inject_sp_noise(O.synth_image(W, H, G * 7 + W), 0.3, 0.5, 11)
    tmax = tmax or lib().phg_max_fused_iterations(beta)
    pitch = (W + 15) // 16 * 16
    params = PhgParams(20, beta, k, 3, border)
    counters = torch.zeros((k, 2), dtype=torch.int64, device="cuda")
    plans = [D.BandPlan(H, W, G, r, beta * tmax) for r in range(G)]
    bufs = []
    for p in plans:
        b = [torch.zeros((p.rows, pitch), dtype=torch.uint8, device="cuda") for _ in range(3)]
        b[0][:, :W] = torch.from_numpy(img[p.blo:p.bhi]).cuda()
        bufs.append(b)
    step = D.cuda_band_stepper(params, counters, W, H)
    cur = [b[0] for b in bufs]
    nxt = [b[1] for b in bufs]
    for it0_iters in [(sum(D.chunk_plan(k, tmax)[:i]), n) for i, n in enumerate(D.chunk_plan(k, tmax))]:
        it0, iters = it0_iters
        for p, s, d in zip(plans, cur, nxt):
            step(s, d, p, it0, iters)
        for i, p in enumerate(plans):  # halo exchange as device copies
            if p.up is not None:
                q = plans[p.up]
                nxt[i][0:p.lo - p.blo] = nxt[p.up][q.local(p.blo):q.local(p.lo)]
            if p.down is not None:
                q = plans[p.down]
                nxt[i][p.local(p.hi):p.rows] = nxt[p.down][q.local(p.hi):q.local(p.bhi)]
        for i in range(G):
            spare = [b for b in bufs[i] if b is not cur[i] and b is not nxt[i]][0]
            cur[i], nxt[i] = nxt[i], spare
    torch.cuda.synchronize()
    out = np.concatenate([c[p.local(p.lo):p.local(p.hi), :W].cpu().numpy() for p, c in zip(plans, cur)])
    ref, ref_stats = O.denoise(img, 20, beta, k, 3, border)
    assert np.array_equal(out, ref)
    assert D.truncate_stats(counters.cpu()) == ref_stats
