"""GPU parity of the beta = 2 kernel on both integer pipes (fused_h2b2_kernel,
kernel_h2b2.cuh), which runs every beta=2 / Faithful / card_threshold <= 3
denoise (C3).  Bit-exact image and per-iteration stats against the oracle
(denoise.hpp:292-311).  Edge cases specific to its design:
  - the sweep ignores the image edges and border pixels (within 2 of an
    edge) are counted by the scalar border pass: images smaller than the
    window, 1-4 px strips, widths/heights around the 496-px tile;
  - the two fp16 lanes hold different images / tiles (batches, odd tile
    counts);
  - alpha > 128 (the AND form of the byte-SIMD carry test) and alpha = 1;
  - dense candidates (uniform random images) for the two-per-lane drain;
  - k split into launches of T <= 4 (k = 1..9).
"""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(noisy, alpha=20, k=5, thr=3):
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams(alpha, 2, k, thr))
    ref_img, ref_stats = O.denoise(noisy, alpha, 2, k, thr, 0)
    assert np.array_equal(res.image.pixels, ref_img), (noisy.shape, alpha, k, thr)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats


def test_kernel_selected():
    assert P.kernel_name(P.DenoiseParams(beta=2), 4) == "fused_bp2_kernel<T=4>"
    assert P.kernel_name(P.DenoiseParams(beta=2, card_threshold=3), 2) == "fused_bp2_kernel<T=2>"
    assert P.kernel_name(P.DenoiseParams(beta=2, card_threshold=4), 4).startswith("fused_tb_kernel")


@pytest.mark.parametrize("alpha", [1, 2, 20, 127, 128, 129, 200, 255])
def test_uniform_random_dense_candidates(alpha):
    rng = np.random.default_rng(alpha)
    _check(rng.integers(0, 256, (150, 1010), dtype=np.uint8), alpha=alpha)


@pytest.mark.parametrize("density", [0.05, 0.3, 0.5, 0.7, 1.0])
def test_salt_and_pepper_densities(density):
    clean = O.synth_image(700, 300, 5)
    _check(O.inject_sp_noise(clean, density, 0.5, 17))


@pytest.mark.parametrize("thr", [1, 2, 3])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 9])
def test_thresholds_and_chunks(thr, k):
    clean = O.synth_image(530, 97, 10 * thr + k)
    _check(O.inject_sp_noise(clean, 0.45, 0.4, k), k=k, thr=thr)


@pytest.mark.parametrize("w,h", [(1, 1), (2, 7), (4, 4), (5, 5), (6, 3), (3, 60), (40, 2), (16, 40), (481, 37),
                                 (495, 20), (496, 73), (497, 36), (992, 31), (993, 45), (1489, 29), (2000, 6)])
def test_tile_geometry_and_small_images(w, h):
    clean = O.synth_image(w, h, w * 3 + h)
    _check(O.inject_sp_noise(clean, 0.35, 0.5, 3))


@pytest.mark.parametrize("n,h", [(2, 40), (3, 37), (5, 101)])
def test_batch_lanes_span_images(n, h):
    w = 481
    imgs = np.stack([O.inject_sp_noise(O.synth_image(w, h, 200 + i), 0.1 + 0.15 * i, 0.5, i) for i in range(n)])
    out, stats = P.denoise_batch(imgs, P.DenoiseParams(beta=2))
    for i in range(n):
        ref, st = O.denoise(imgs[i], 20, 2, 5, 3, 0)
        assert np.array_equal(out[i], ref), i
        assert [(s.flagged, s.replaced) for s in stats[i]] == st


def test_bands_and_tb_agree():
    # the same image through h2b2 (Faithful) in row bands, and the byte-SIMD
    # kernel forced by InBounds on a threshold where both borders agree on nothing
    img = O.inject_sp_noise(O.synth_image(900, 260, 8), 0.4, 0.5, 2)
    ref, ref_st = O.denoise(img, 20, 2, 7, 3, 0)
    res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(20, 2, 7, 3), P.EngineSpec.parallel(3))
    assert np.array_equal(res.image.pixels, ref)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_st
