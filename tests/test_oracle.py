"""The oracle (oracle/phgrms_oracle.c) pinned against the reference: its own
hand-derived vectors (proj/tests/test_denoise.cpp, test_noise.cpp,
acceptance.cpp crit 3) and fixtures produced by running the reference itself
(tests/golden/, made by tests/golden/make_golden.py).  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_small():
    z = np.load(os.path.join(GOLD, "small_cases.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    for i, m in enumerate(meta):
        yield m, z[f"img_{i}"], z[f"card_{i}"], z[f"pass_out_{i}"], z[f"final_{i}"]


# ------------------------------------------------ reference hand-derived KATs
def test_kat_cardinality_3x3():
    assert O.cardinality(np.full((3, 3), 100, np.uint8), 20, 1).ravel().tolist() == [4, 6, 4, 6, 9, 6, 4, 6, 4]
    img = np.full((3, 3), 100, np.uint8)
    img[1, 1] = 255
    assert O.cardinality(img, 20, 1).ravel().tolist() == [3, 5, 3, 5, 1, 5, 3, 5, 3]
    for a in (1, 20, 255):
        assert O.cardinality(np.full((1, 1), 42, np.uint8), a, 1).tolist() == [[1]]


def test_kat_removal_and_border_fork():
    img = np.full((3, 3), 100, np.uint8)
    img[1, 1] = 255
    out, f, r = O.removal_pass(img, O.cardinality(img, 20, 1))
    assert (out == 100).all() and (f, r) == (1, 1)
    img = np.full((4, 4), 50, np.uint8)
    img[0, 0] = 255
    card = O.cardinality(img, 20, 1)
    kept, f, r = O.removal_pass(img, card, border=0)
    assert (kept == img).all() and (f, r) == (1, 0)
    fixed, f, r = O.removal_pass(img, card, border=1)
    assert (fixed == 50).all() and r == 1


def test_kat_two_impulses_and_fixed_point():
    img = np.full((7, 7), 100, np.uint8)
    img[3, 3] = img[3, 4] = 255
    out, st = O.denoise(img)
    assert (out == 100).all() and [r for _, r in st] == [2, 0]
    out, st = O.denoise(np.full((64, 64), 77, np.uint8))
    assert len(st) == 1 and st[0][1] == 0


def test_kat_replaced_but_unchanged():
    img = np.array([[0, 141, 0], [141, 100, 141], [0, 141, 0]], np.uint8)
    out, st = O.denoise(img, k=3)
    assert (out == img).all() and [r for _, r in st] == [1, 1, 1]


def test_kat_rms_replacement():
    # test_denoise.cpp:267-275
    assert [O.rms_replacement(s, f) for s, f in [(0, 1), (2, 1), (9, 4), (25, 4), (65025, 1), (65025 * 8, 8)]] == \
        [0, 1, 2, 3, 255, 255]


def test_kat_mt19937_and_noise_seed77():
    # C++ [rand.predef]: the 10000th output of a default-seeded mt19937 is 4123659995
    assert O.lib().orc_mt19937_nth(5489, 10000) == 4123659995
    noisy, mask = O.inject_sp_noise(np.full((10, 10), 100, np.uint8), 0.2, 0.5, 77, with_mask=True)
    salt = {4, 13, 14, 22, 47, 55, 64, 65, 90, 96}
    pepper = {2, 16, 18, 24, 41, 42, 68, 70, 73, 77}
    flat, m = noisy.ravel(), mask.ravel()
    for i in range(100):
        exp = 255 if i in salt else 0 if i in pepper else 100
        assert flat[i] == exp and m[i] == (i in salt or i in pepper)
    _, mask = O.inject_sp_noise(np.full((10, 10), 128, np.uint8), 0.505, 0.5, 5, with_mask=True)
    assert mask.sum() == 51


def test_kat_row_blocks():
    for h in (0, 1, 2, 5, 7, 64, 1000):
        for wk in (1, 2, 3, 8, 64):
            b = O.row_blocks(h, wk)
            assert len(b) <= min(h, wk) and sum(e - s for s, e in b) == h
            assert all(e > s for s, e in b) and all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
    assert len(O.row_blocks(5, 8)) == 5


# ------------------------------------------------------ vs the reference run
def test_small_cases_match_reference_fixtures():
    n = 0
    for m, img, card, pass_out, final in load_small():
        n += 1
        a, b, k, thr, border = m["alpha"], m["beta"], m["k"], m["thr"], m["border"]
        assert np.array_equal(O.cardinality(img, a, b), card)
        out, f, r = O.removal_pass(img, card, a, b, thr, border)
        assert np.array_equal(out, pass_out) and [f, r] == m["pass_stats"]
        fin, st = O.denoise(img, a, b, k, thr, border)
        assert np.array_equal(fin, final) and [list(x) for x in st] == m["stats"]
    assert n == 80


def test_generators_and_c1_match_reference_digests():
    d = json.load(open(os.path.join(GOLD, "digests.json")))
    c1 = d["c1"]
    clean = O.synth_image(481, 321, 1)
    noisy = O.inject_sp_noise(clean, 0.10, 0.5, 12345)
    assert sha(clean) == c1["clean"] and sha(noisy) == c1["noisy"]
    assert sha(O.cardinality(noisy, 20, 1)) == c1["card1"]
    fin, st = O.denoise(noisy)
    assert sha(fin) == c1["final"] and [list(x) for x in st] == c1["stats"]
    fin64, st64 = O.denoise(noisy, k=64)
    assert sha(fin64) == c1["final_k64"] and [list(x) for x in st64] == c1["stats_k64"]
    flat = O.inject_sp_noise(np.full((321, 481), 128, np.uint8), 0.01, 0.5, 7)
    fin, st = O.denoise(flat)
    assert sha(fin) == d["flat_1pct"]["final"] and [list(x) for x in st] == d["flat_1pct"]["stats"]
    assert [r for _, r in st] == [1526, 25, 0]


def test_c4_first_images_match_reference_digests():
    d = json.load(open(os.path.join(GOLD, "digests.json")))["c4_first16"]
    for e in d[:6]:
        n = O.inject_sp_noise(O.synth_image(481, 321, e["i"]), e["density"], 0.5, e["i"])
        assert sha(n) == e["noisy"]
        fin, st = O.denoise(n)
        assert sha(fin) == e["final"] and [list(x) for x in st] == e["stats"]


def test_period_two_cycle():
    # 481x321 at 10% settles into an exact period-2 cycle
    n = O.inject_sp_noise(O.synth_image(481, 321, 3), 0.10, 0.5, 99)
    imgs = [O.denoise(n, k=k)[0] for k in (50, 51, 52)]
    assert np.array_equal(imgs[0], imgs[2]) and not np.array_equal(imgs[0], imgs[1])


@pytest.mark.skipif(not O.ref_available(), reason="reference not compiled here")
def test_oracle_equals_reference_live():
    """Where the reference library is present, compare live on fresh seeds
    (including the paper's scatter form of Algorithm 1)."""
    rng = np.random.default_rng(5)
    R = O.ref()
    for _ in range(40):
        w, h = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        a, b = int(rng.integers(1, 256)), int(rng.integers(1, 4))
        assert np.array_equal(O.cardinality(img, a, b), O.ref_cardinality(img, a, b))
        assert np.array_equal(O.cardinality_scatter(img, a, b), O.cardinality(img, a, b))
        for border in (0, 1):
            x, sx = O.denoise(img, a, b, 5, 3, border)
            y, sy = O.ref_denoise(img, a, b, 5, 3, border, workers=3)
            assert np.array_equal(x, y) and sx == sy


def test_band_pass_equals_full_image():
    """orc_band_pass over any row split reproduces one full-image pass."""
    rng = np.random.default_rng(9)
    img = O.inject_sp_noise(O.synth_image(57, 41, 2), 0.3, 0.5, 3)
    for beta in (1, 2):
        full, f, r = O.removal_pass(img, O.cardinality(img, 20, beta), 20, beta)
        out = np.empty_like(img)
        tf = tr = 0
        for lo, hi in O.row_blocks(41, 4):
            blo, bhi = max(0, lo - beta), min(41, hi + beta)
            band = np.ascontiguousarray(img[blo:bhi])
            bout = band.copy()
            ff, rr = O.band_pass(band, bout, blo, 41, lo, hi, lo, hi, 20, beta)
            out[lo:hi] = bout[lo - blo:hi - blo]
            tf, tr = tf + ff, tr + rr
        assert np.array_equal(out, full) and (tf, tr) == (f, r)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_band_wise_reference_equals_whole_image():
    """Pins the method behind the C5 golden digest (tests/golden/make_golden.py
    c5_full): k reference passes on row bands with a beta*k-row halo give the
    whole-image reference's image, and the owned-row counters sum to its
    per-iteration stats."""
    img = O.ref_inject_sp_noise(O.ref_synth_image(700, 333, 4), 0.3, 0.5, 8)
    fin, st = O.ref_denoise(img)
    parts, tot = [], np.zeros((5, 2), np.int64)
    for lo in range(0, 333, 50):
        hi = min(333, lo + 50)
        blo, bhi = max(0, lo - 5), min(333, hi + 5)
        out, bst = O.ref_denoise_band(img[blo:bhi], lo - blo, hi - blo)
        parts.append(out)
        tot += np.array(bst, np.int64)
    assert np.array_equal(np.concatenate(parts), fin)
    assert [tuple(int(x) for x in r) for r in tot[:len(st)]] == st
