"""phg_denoise_sharded (the Parallel engine with GPUs as workers, one
process driving every listed device) on one B200: device lists that repeat
device 0 run the same band/halo schedule -- per-band buffers, halo rows
copied with cudaMemcpyPeerAsync after every fused launch, per-device
counters summed on the host -- as a multi-GPU list, so the results must be
bit-identical to the full-image oracle (denoise.hpp:292-311)."""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ndev,W,H,beta,k,thr,border", [
    (1, 481, 321, 1, 5, 3, 0), (2, 481, 321, 1, 5, 3, 0), (3, 700, 257, 2, 5, 3, 1),
    (4, 1000, 200, 1, 7, 3, 0), (5, 333, 90, 3, 3, 4, 0), (8, 520, 400, 1, 12, 2, 1),
    (16, 300, 40, 1, 5, 3, 0),  # bands of 2-3 rows: halos reach past the neighbour
])
def test_single_image_bands_equal_full_image(ndev, W, H, beta, k, thr, border):
    img = O.inject_sp_noise(O.synth_image(W, H, ndev * 13 + W), 0.3, 0.5, 5)
    params = P.DenoiseParams(20, beta, k, thr, P.BorderMode(border))
    out, stats = P.denoise_sharded(img, params, [0] * ndev)
    ref, ref_stats = O.denoise(img, 20, beta, k, thr, border)
    assert np.array_equal(out, ref)
    assert [(s.flagged, s.replaced) for s in stats] == ref_stats
    assert [s.iteration for s in stats] == list(range(1, len(ref_stats) + 1))


def test_single_image_early_stop():
    flat = np.full((321, 481), 128, np.uint8)
    noisy = O.inject_sp_noise(flat, 0.01, 0.5, 7)
    _, stats = P.denoise_sharded(noisy, P.DenoiseParams(), [0, 0, 0])
    assert [s.replaced for s in stats] == [1526, 25, 0]


@pytest.mark.parametrize("n,ndev", [(2, 1), (5, 2), (7, 3), (3, 8)])
def test_batch_shards_equal_per_image(n, ndev):
    w, h = 300, 77
    imgs = np.stack([O.inject_sp_noise(O.synth_image(w, h, 40 + i), 0.05 + 0.1 * i, 0.5, i) for i in range(n)])
    out, stats = P.denoise_sharded(imgs, P.DenoiseParams(), [0] * ndev)
    for i in range(n):
        ref, st = O.denoise(imgs[i])
        assert np.array_equal(out[i], ref), i
        assert [(s.flagged, s.replaced) for s in stats[i]] == st


def test_bad_device_rejected():
    with pytest.raises(P.InvalidArgument, match="does not exist"):
        P.denoise_sharded(np.zeros((8, 8), np.uint8), P.DenoiseParams(), [0, 4096])


@pytest.mark.parametrize("ndev,beta,k", [(3, 1, 5), (4, 2, 9), (2, 3, 2)])
def test_copy_exchange_equals_peer_stores(monkeypatch, ndev, beta, k):
    # bands >= one halo tall use the kernels' peer stores; PHG_SHARD_COPY=1
    # forces the copy exchange on the same split -- both equal the oracle
    img = O.inject_sp_noise(O.synth_image(600, 211, 77 + beta), 0.25, 0.5, 3)
    params = P.DenoiseParams(20, beta, k, 3)
    ref, ref_stats = O.denoise(img, 20, beta, k, 3, 0)
    peer, st_peer = P.denoise_sharded(img, params, [0] * ndev)
    monkeypatch.setenv("PHG_SHARD_COPY", "1")
    copy, st_copy = P.denoise_sharded(img, params, [0] * ndev)
    assert np.array_equal(peer, ref) and np.array_equal(copy, ref)
    assert [(s.flagged, s.replaced) for s in st_peer] == ref_stats
    assert [(s.flagged, s.replaced) for s in st_copy] == ref_stats
