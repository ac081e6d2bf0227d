"""beta = 3 on the temporally blocked byte-SIMD kernel (fused_tb_kernel<3, T<=2>):
7x7 windows, halo 3T rows/columns.  Bit-exact image and per-iteration stats
against the oracle (denoise.hpp:292-311) across borders, thresholds (flag
bound pix_count - 3 = 46 for Faithful), iteration chunking, tile geometry and
row bands.  Before this kernel, beta >= 3 ran the one-pixel-per-thread
scalar kernel, one launch per iteration."""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(noisy, alpha=20, k=5, thr=3, border=0, bands=1):
    eng = P.EngineSpec.parallel(bands) if bands > 1 else P.EngineSpec.serial()
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams(alpha, 3, k, thr, P.BorderMode(border)), eng)
    ref_img, ref_stats = O.denoise(noisy, alpha, 3, k, thr, border)
    assert np.array_equal(res.image.pixels, ref_img), (noisy.shape, alpha, k, thr, border)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats


def test_kernel_selected():
    assert P.lib().phg_max_fused_iterations(3) == 2
    assert P.kernel_name(P.DenoiseParams(beta=3), 2) == "fused_tb_kernel<beta=3,T=2>"
    assert P.kernel_name(P.DenoiseParams(beta=3), 3) == ""
    assert P.kernel_name(P.DenoiseParams(beta=4), 1) == "scalar_kernel<fused>"


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("border", [0, 1])
def test_iteration_chunks_and_borders(k, border):
    noisy = O.inject_sp_noise(O.synth_image(530, 151, k + 10 * border), 0.4, 0.5, k)
    _check(noisy, k=k, border=border)


@pytest.mark.parametrize("thr", [1, 2, 5, 13, 30, 49, 50, 1000])
def test_thresholds(thr):
    noisy = O.inject_sp_noise(O.synth_image(300, 120, thr), 0.5, 0.5, 2)
    _check(noisy, thr=thr, border=thr % 2)


@pytest.mark.parametrize("alpha", [1, 7, 60, 128, 129, 255])
def test_alpha_and_dense_noise(alpha):
    rng = np.random.default_rng(alpha)
    _check(rng.integers(0, 256, (97, 700), dtype=np.uint8), alpha=alpha)


@pytest.mark.parametrize("w,h", [(1, 1), (3, 9), (7, 7), (8, 3), (495, 14), (496, 64), (497, 65), (993, 33),
                                 (2000, 5)])
def test_tile_geometry(w, h):
    noisy = O.inject_sp_noise(O.synth_image(w, h, w * 7 + h), 0.3, 0.5, 1)
    _check(noisy)
    _check(noisy, border=1, k=3)


@pytest.mark.parametrize("bands", [2, 5])
def test_row_bands(bands):
    noisy = O.inject_sp_noise(O.synth_image(640, 200, 3), 0.3, 0.5, 9)
    _check(noisy, k=6, bands=bands)
