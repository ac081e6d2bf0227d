"""GPU parity of the two-tile fp16 kernel (fused_h2_kernel, kernel_h2.cuh),
which runs every beta=1 / Faithful / card_threshold <= 3 denoise.

Edge cases specific to its design, each checked bit-exactly (image and
per-iteration stats) against the oracle restating denoise.hpp:292-311:
  - the B lane of the last CTA is empty (odd tile counts) and the two lanes
    of one CTA belong to different images / column tiles;
  - dense candidate rows (uniform-random images: ~2/3 of the pixels are
    candidates) exercise the warp ring at its largest quads;
  - card_threshold 1 and 2 (candidate threshold m = thr - 2);
  - widths around the 496-px tile, heights around the tile plan.
"""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(noisy, alpha=20, k=5, thr=3):
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams(alpha, 1, k, thr))
    ref_img, ref_stats = O.denoise(noisy, alpha, 1, k, thr, 0)
    assert np.array_equal(res.image.pixels, ref_img), (noisy.shape, alpha, k, thr)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats


def test_kernel_selected():
    L = P.lib()
    assert P.kernel_name(P.DenoiseParams(), 5) == "fused_bp_kernel<T=5>"
    assert P.kernel_name(P.DenoiseParams(card_threshold=4), 5).startswith("fused_tb_kernel")
    assert P.kernel_name(P.DenoiseParams(beta=2), 4) == "fused_bp2_kernel<T=4>"
    assert P.kernel_name(P.DenoiseParams(beta=2, border=P.BorderMode(1)), 4).startswith("fused_tb_kernel")
    assert P.kernel_name(P.DenoiseParams(beta=2, card_threshold=4), 4).startswith("fused_tb_kernel")
    assert L is not None


@pytest.mark.parametrize("alpha", [1, 5, 20, 128, 129, 255])
def test_uniform_random_images_dense_candidates(alpha):
    rng = np.random.default_rng(alpha)
    img = rng.integers(0, 256, (173, 1100), dtype=np.uint8)
    _check(img, alpha=alpha)


@pytest.mark.parametrize("density", [0.7, 0.9, 1.0])
def test_heavy_salt_and_pepper(density):
    clean = O.synth_image(640, 480, 11)
    noisy = O.inject_sp_noise(clean, density, 0.5, 21)
    _check(noisy)


@pytest.mark.parametrize("thr", [1, 2, 3])
@pytest.mark.parametrize("k", [1, 3, 5, 7, 12])
def test_thresholds_and_iteration_chunks(thr, k):
    clean = O.synth_image(530, 97, thr * 10 + k)
    noisy = O.inject_sp_noise(clean, 0.35, 0.4, k)
    _check(noisy, k=k, thr=thr)


@pytest.mark.parametrize("w,h", [(3, 3), (16, 40), (481, 36), (481, 37), (496, 73), (497, 36),
                                 (992, 31), (993, 45), (1489, 29), (2000, 7)])
def test_tile_geometry(w, h):
    clean = O.synth_image(w, h, w + h)
    noisy = O.inject_sp_noise(clean, 0.25, 0.5, 3)
    _check(noisy)


@pytest.mark.parametrize("n,h", [(1, 321), (3, 36), (5, 37), (7, 100)])
def test_batch_lanes_span_images(n, h):
    # consecutive tiles -- possibly of different images -- share one CTA
    w = 481
    imgs = np.empty((n, h, w), np.uint8)
    for i in range(n):
        imgs[i] = O.inject_sp_noise(O.synth_image(w, h, 100 + i), 0.1 + 0.15 * i, 0.5, i)
    out, stats = P.denoise_batch(imgs, P.DenoiseParams())
    for i in range(n):
        ref, st = O.denoise(imgs[i])
        assert np.array_equal(out[i], ref), i
        assert [(s.flagged, s.replaced) for s in stats[i]] == st


def test_flat_image_stops_early_through_h2():
    # constant 128 + 1% noise stops at iteration 3 (SURVEY.md 8(c) KAT)
    flat = np.full((321, 481), 128, np.uint8)
    noisy = O.inject_sp_noise(flat, 0.01, 0.5, 7)
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams())
    assert [s.replaced for s in res.stats] == [1526, 25, 0]
    ref_img, _ = O.denoise(noisy)
    assert np.array_equal(res.image.pixels, ref_img)


@pytest.mark.parametrize("beta,k,border", [(1, 5, 0), (1, 12, 0), (2, 5, 0), (2, 9, 1), (3, 2, 0)])
def test_row_pipelined_single_image(beta, k, border):
    # images >= 32 MB go host -> device -> host in row chunks (denoise_rows_pipelined)
    clean = O.synth_image(4096, 8193, 31 + beta)
    noisy = O.inject_sp_noise(clean, 0.4, 0.5, 7 + k)
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams(20, beta, k, 3, P.BorderMode(border)))
    ref_img, ref_stats = O.denoise(noisy, 20, beta, k, 3, border)
    assert np.array_equal(res.image.pixels, ref_img)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats
    out, stats = P.denoise_batch(noisy[None], P.DenoiseParams(20, beta, k, 3, P.BorderMode(border)))
    assert np.array_equal(out[0], ref_img)
    assert [(s.flagged, s.replaced) for s in stats[0]] == ref_stats
