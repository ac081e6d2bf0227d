"""beta >= 4 (the scalar fused kernel, one launch per iteration) against the
oracle, and the row-pipelined single-image path with halos taller than its
chunks (a 16384x300 image at beta=120 used to get 100-row chunks
under a 120-row halo).

The reference accepts any beta >= 1 (denoise.hpp:41-49); every case is
bit-exact in the image and the per-iteration (flagged, replaced) stats.
"""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(img, beta, k, border=0, thr=3, alpha=20, bands=1):
    eng = P.EngineSpec.parallel(bands) if bands > 1 else P.EngineSpec.serial()
    res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(alpha, beta, k, thr, P.BorderMode(border)), eng)
    ref_img, ref_stats = O.denoise(img, alpha, beta, k, thr, border)
    assert np.array_equal(res.image.pixels, ref_img), (img.shape, beta, k, border, bands)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, (img.shape, beta, k, border, bands)


@pytest.mark.parametrize("beta", [4, 5, 7])
@pytest.mark.parametrize("border", [0, 1])
@pytest.mark.parametrize("k", [1, 3])
def test_beta_ge4_small(beta, border, k):
    img = O.inject_sp_noise(O.synth_image(97, 61, beta + 10 * k), 0.3, 0.5, border + 3)
    _check(img, beta, k, border, thr=beta * beta)


@pytest.mark.parametrize("beta,bands", [(4, 3), (7, 2), (5, 4)])
def test_beta_ge4_row_bands(beta, bands):
    img = O.inject_sp_noise(O.synth_image(120, 90, beta), 0.4, 0.5, 11)
    _check(img, beta, 3, 0, thr=2 * beta, bands=bands)


@pytest.mark.parametrize("beta,k", [(4, 3), (7, 2)])
def test_beta_ge4_pipelined_image(beta, k):
    # >= 4 MB: the row-pipelined host path (chunks of copies and launches)
    img = O.inject_sp_noise(O.synth_image(4096, 1100, beta), 0.3, 0.5, 5)
    _check(img, beta, k, 0, thr=beta * beta)


def test_pipelined_chunks_never_shorter_than_the_halo(monkeypatch):
    # eight 32-row chunks under a 33-row halo: the plan must use taller chunks
    monkeypatch.setenv("PHG_ROW_CHUNKS", "8")
    img = O.inject_sp_noise(O.synth_image(1024, 256, 3), 0.3, 0.5, 9)
    _check(img, 33, 2, 0, thr=400)
    _check(img, 2, 9, 0)   # beta * T = 2 * 5 rows
    _check(img, 1, 12, 0)
