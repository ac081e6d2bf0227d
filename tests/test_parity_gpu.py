"""GPU parity: the sm_100a path (through the C ABI) vs the oracle, bit-exact.

Mirrors the reference's own hot-path tests (proj/tests/test_denoise.cpp,
test_parallel.cpp, acceptance.cpp criteria 1-3) plus the BASELINE configs.
"""
import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

G = P.GrayImage


def _img(a):
    return G.from_array(np.asarray(a, np.uint8))


def _params(alpha=20, beta=1, k=5, thr=3, border=0):
    return P.DenoiseParams(alpha, beta, k, thr, P.BorderMode(border))


def _check_denoise(noisy, alpha=20, beta=1, k=5, thr=3, border=0, bands=1):
    eng = P.EngineSpec.serial() if bands <= 1 else P.EngineSpec.parallel(bands)
    res = P.denoise(_img(noisy), _params(alpha, beta, k, thr, border), eng)
    ref_img, ref_stats = O.denoise(noisy, alpha, beta, k, thr, border)
    assert np.array_equal(res.image.pixels, ref_img), (alpha, beta, k, thr, border, bands)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats
    assert [s.iteration for s in res.stats] == list(range(1, len(ref_stats) + 1))


# ------------------------------------------------ test_denoise.cpp fixtures
def test_cardinality_constant_3x3():
    card = P.compute_cardinality(G(3, 3, 100), 20, 1)
    assert card.counts.tolist() == [4, 6, 4, 6, 9, 6, 4, 6, 4]


def test_cardinality_impulse_3x3():
    img = G(3, 3, 100)
    img.set(1, 1, 255)
    assert P.compute_cardinality(img, 20, 1).counts.tolist() == [3, 5, 3, 5, 1, 5, 3, 5, 3]


@pytest.mark.parametrize("alpha", [1, 20, 255])
def test_cardinality_single_pixel(alpha):
    assert P.compute_cardinality(G(1, 1, 42), alpha, 1).counts.tolist() == [1]


def test_removal_restores_impulse():
    img = G(3, 3, 100)
    img.set(1, 1, 255)
    card = P.compute_cardinality(img, 20, 1)
    out, st = P.denoise_pass(img, card, P.DenoiseParams())
    assert out == G(3, 3, 100) and st.flagged == 1 and st.replaced == 1


def test_border_mode_fork():
    img = G(4, 4, 50)
    img.set(0, 0, 255)
    card = P.compute_cardinality(img, 20, 1)
    assert card.at(0, 0) == 1
    kept, ks = P.denoise_pass(img, card, P.DenoiseParams())
    assert kept == img and ks.flagged == 1 and ks.replaced == 0
    fixed, fs = P.denoise_pass(img, card, P.DenoiseParams(border=P.BorderMode.InBounds))
    assert fixed == G(4, 4, 50) and fs.replaced == 1


def test_two_adjacent_impulses():
    img = G(7, 7, 100)
    img.set(3, 3, 255)
    img.set(3, 4, 255)
    card = P.compute_cardinality(img, 20, 1)
    assert card.at(3, 3) == 2 and card.at(3, 4) == 2
    res = P.denoise(img, P.DenoiseParams())
    assert res.image == G(7, 7, 100)
    assert [s.replaced for s in res.stats] == [2, 0]


def test_constant_image_stops_after_one_pass():
    res = P.denoise(G(64, 64, 77), P.DenoiseParams())
    assert res.image == G(64, 64, 77)
    assert len(res.stats) == 1 and res.stats[0].iteration == 1 and res.stats[0].replaced == 0


@pytest.mark.parametrize("beta", [1, 2, 3])
def test_removal_leaves_constant_untouched(beta):
    p = P.DenoiseParams(beta=beta)
    img = G(6, 5, 200)
    out, st = P.denoise_pass(img, P.compute_cardinality(img, p.alpha, p.beta), p)
    assert out == img and st.flagged == 0 and st.replaced == 0


def test_replaced_but_unchanged_keeps_iterating():
    # replaced != "pixel changed"
    img = _img([[0, 141, 0], [141, 100, 141], [0, 141, 0]])
    res = P.denoise(img, P.DenoiseParams(max_iterations=3))
    assert res.image == img
    assert [s.replaced for s in res.stats] == [1, 1, 1]


def test_parameter_validation_messages():
    img = G(4, 4, 1)
    for kw, msg in [({"alpha": 0}, "alpha must be in [1, 255]"), ({"alpha": 256}, "alpha must be in [1, 255]"),
                    ({"beta": 0}, "beta must be >= 1"), ({"max_iterations": 0}, "iterations must be >= 1"),
                    ({"card_threshold": 0}, "card_threshold must be >= 1")]:
        with pytest.raises(P.InvalidArgument, match=msg.replace("[", r"\[").replace("]", r"\]")):
            P.denoise(img, P.DenoiseParams(**kw))
    card = P.compute_cardinality(G(3, 3, 1), 20, 1)
    with pytest.raises(P.InvalidArgument, match="cardinality map does not match image"):
        P.denoise_pass(img, card, P.DenoiseParams())


# --------------------------------------------- randomized vs the oracle
def test_cardinality_random_vs_oracle():
    rng = np.random.default_rng(100)
    for _ in range(120):
        w, h = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        alpha, beta = int(rng.integers(1, 256)), int(rng.integers(1, 4))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = P.compute_cardinality(_img(img), alpha, beta).counts.reshape(h, w)
        assert np.array_equal(got, O.cardinality(img, alpha, beta)), (w, h, alpha, beta)


def test_removal_random_vs_oracle():
    rng = np.random.default_rng(102)
    for _ in range(120):
        w, h = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        alpha, beta = int(rng.integers(1, 256)), int(rng.integers(1, 4))
        thr, border = int(rng.choice([1, 2, 3, 4, 7, 30])), int(rng.integers(0, 2))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        card = O.cardinality(img, alpha, beta)
        if rng.integers(0, 3) == 0:  # arbitrary caller-supplied maps are honoured
            card = rng.integers(0, 10, (h, w)).astype(np.int32)
        p = _params(alpha, beta, 1, thr, border)
        out, st = P.denoise_pass(_img(img), P.CardinalityMap(w, h, card.reshape(-1)), p)
        ref, f, r = O.removal_pass(img, card, alpha, beta, thr, border)
        assert np.array_equal(out.pixels, ref) and (st.flagged, st.replaced) == (f, r)


@pytest.mark.parametrize("beta", [1, 2, 3])
def test_denoise_random_small_vs_oracle(beta):
    rng = np.random.default_rng(20240501 + beta)
    for _ in range(60):
        w, h = int(rng.integers(1, 49)), int(rng.integers(1, 49))
        alpha = int(rng.integers(1, 61))
        k = int(rng.choice([1, 5, 8]))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        for border in (0, 1):
            _check_denoise(img, alpha, beta, k, 3, border)


def test_denoise_alpha_and_threshold_sweep():
    rng = np.random.default_rng(7)
    clean = O.synth_image(200, 150, 3)
    for alpha in (1, 2, 19, 20, 64, 127, 128, 129, 200, 255):
        for thr in (1, 3, 5, 10, 26, 1000):
            noisy = O.inject_sp_noise(clean, float(rng.uniform(0.05, 0.6)), 0.5, int(rng.integers(0, 2**31)))
            _check_denoise(noisy, alpha, 1, 5, thr, int(rng.integers(0, 2)))


@pytest.mark.parametrize("w,h", [(1, 300), (300, 1), (2, 2), (5, 1000), (495, 17), (496, 9), (497, 70),
                                 (511, 64), (512, 65), (1000, 3), (993, 130)])
@pytest.mark.parametrize("beta", [1, 2])
def test_ragged_shapes(w, h, beta):
    clean = O.synth_image(w, h, w * 7 + h)
    noisy = O.inject_sp_noise(clean, 0.3, 0.5, 99)
    for border in (0, 1):
        _check_denoise(noisy, 20, beta, 5, 3, border)


# ------------------------------------------------------- partition invariance
@pytest.mark.parametrize("band_engine", [False, True])
@pytest.mark.parametrize("bands", [2, 3, 8])
def test_parallel_bands_equal_serial(bands, band_engine, monkeypatch):
    # default: Parallel(W) runs the single-image pipeline; PHG_BAND_ENGINE=1
    # runs W row bands with halo exchange on the device
    if band_engine:
        monkeypatch.setenv("PHG_BAND_ENGINE", "1")
    rng = np.random.default_rng(201)
    for _ in range(25):
        w, h = int(rng.integers(1, 33)), int(rng.integers(1, 33))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        alpha, beta, border = int(rng.integers(1, 61)), int(rng.integers(1, 3)), int(rng.integers(0, 2))
        _check_denoise(img, alpha, beta, 5, 3, border, bands=bands)


@pytest.mark.parametrize("band_engine", [False, True])
@pytest.mark.parametrize("bands", [2, 5, 16])
def test_parallel_bands_large(bands, band_engine, monkeypatch):
    if band_engine:
        monkeypatch.setenv("PHG_BAND_ENGINE", "1")
    clean = O.synth_image(700, 555, 5)
    noisy = O.inject_sp_noise(clean, 0.3, 0.5, 5)
    for beta in (1, 2):
        _check_denoise(noisy, 20, beta, 5, 3, 0, bands=bands)


def test_scatter_equals_gather_on_gpu():
    rng = np.random.default_rng(20240502)
    for _ in range(120):
        w, h = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        alpha, beta = int(rng.integers(1, 61)), int(rng.integers(1, 3))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = P.compute_cardinality(_img(img), alpha, beta).counts.reshape(h, w)
        assert np.array_equal(got, O.cardinality_scatter(img, alpha, beta))


# -------------------------------------------------------- BASELINE configs
def test_config_c1_bsds():
    clean = O.synth_image(481, 321, 1)
    noisy = O.inject_sp_noise(clean, 0.10, 0.5, 12345)
    _check_denoise(noisy)
    _check_denoise(noisy, k=64)


def test_config_c2_4k():
    clean = O.synth_image(3840, 2160, 1)
    noisy = O.inject_sp_noise(clean, 0.30, 0.5, 12345)
    _check_denoise(noisy)
    card = P.compute_cardinality(_img(noisy), 20, 1).counts.reshape(2160, 3840)
    assert np.array_equal(card, O.cardinality(noisy, 20, 1))


def test_config_c3_beta2_crop():
    clean = O.synth_image(2048, 2048, 1)
    noisy = O.inject_sp_noise(clean, 0.50, 0.5, 12345)
    _check_denoise(noisy, beta=2)


def test_config_c4_batch_subset():
    n, w, h = 24, 481, 321
    imgs = np.empty((n, h, w), np.uint8)
    for i in range(n):
        d = 0.10 + 0.60 * (i % 61) / 60
        imgs[i] = O.inject_sp_noise(O.synth_image(w, h, i), d, 0.5, i)
    out, stats = P.denoise_batch(imgs, P.DenoiseParams())
    for i in range(n):
        ref, st = O.denoise(imgs[i])
        assert np.array_equal(out[i], ref), i
        assert [(s.flagged, s.replaced) for s in stats[i]] == st


def test_generators_match_oracle():
    for seed in (0, 1, 77):
        a = P.synth_image(97, 61, seed)
        assert np.array_equal(a.pixels, O.synth_image(97, 61, seed))
        n1 = P.inject_sp_noise(a, P.NoiseSpec(0.3, 0.5, seed))
        assert np.array_equal(n1.pixels, O.inject_sp_noise(a.pixels, 0.3, 0.5, seed))


# ------------------------------------------- device RMS, exhaustive (h2_rms)
def _rms_exact(S, f):
    """u = llround(sqrt(S/f)) (denoise.hpp:163-169) as the integer rule
    max u: (2u-1)^2 f <= 4S (pinned against the reference's double formula
    in tests/test_abi.py)."""
    S = S.astype(np.int64)
    u = np.floor((np.sqrt(4.0 * S / f) + 1.0) / 2.0).astype(np.int64)
    u -= ((u >= 1) & ((2 * u - 1) ** 2 * f > 4 * S)).astype(np.int64)
    u += ((2 * u + 1) ** 2 * f <= 4 * S).astype(np.int64)
    return u


@pytest.mark.parametrize("f", [7, 8, 23, 24])
def test_device_rms_exhaustive(f):
    """Every S the fused kernels can meet (S <= f * 65025: f dissimilar cells
    of at most 255) gives the reference's rounding bit for bit."""
    import ctypes as C
    from paper_1306_5390_b200._lib import lib
    n = f * 65025 + 1
    out = np.empty(n, np.uint32)
    assert lib().phg_debug_rms(f, n, out.ctypes.data_as(C.c_void_p)) == 0
    S = np.arange(n, dtype=np.int64)
    ref = _rms_exact(S, f)
    bad = np.nonzero(out.astype(np.int64) != ref)[0]
    assert bad.size == 0, [(int(s), int(out[s]), int(ref[s])) for s in bad[:8]]
    for s in (0, 1, 2, 3, 4 * f - 1, 4 * f, f * 65025, 12345):
        assert int(out[s]) == O.rms_replacement(s, f), s
