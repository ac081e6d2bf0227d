"""GPU parity of the packed-bit beta=1 kernel (fused_bp_kernel, kernel_bp.cuh),
which runs every beta=1 / Faithful / card_threshold <= 3 denoise.

Edge cases specific to its design, each checked bit-exactly (image and
per-iteration stats) against the oracle restating denoise.hpp:292-311:
  - the three column layouts: two full-width tiles per CTA (width <= 512),
    one full-width tile (513..1024), 992-column tiles with 16-px aprons
    (> 1024), with widths at every layout and strip boundary;
  - row bands of the 8 warps: computed row counts below 8 (empty warps),
    band edges on image borders, one-row bands;
  - dense candidate rows (uniform-random images, alpha 1..255): list rounds,
    leftovers, a whole 1024-px row of candidates;
  - T = 1..5 launches (k = 1..12), card_threshold 1..3;
  - the device early exit (a converged image stops computing, k = 64).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(noisy, alpha=20, k=5, thr=3):
    res = P.denoise(P.GrayImage.from_array(noisy), P.DenoiseParams(alpha, 1, k, thr))
    ref_img, ref_stats = O.denoise(noisy, alpha, 1, k, thr, 0)
    assert np.array_equal(res.image.pixels, ref_img), (noisy.shape, alpha, k, thr)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, (noisy.shape, alpha, k, thr)


def _sp(w, h, seed, density=0.3):
    return O.inject_sp_noise(O.synth_image(w, h, seed), density, 0.5, seed + 1)


def test_kernel_selected():
    assert P.kernel_name(P.DenoiseParams(), 5) == "fused_bp_kernel<T=5>"
    assert P.kernel_name(P.DenoiseParams(card_threshold=2), 3) == "fused_bp_kernel<T=3>"
    assert P.kernel_name(P.DenoiseParams(card_threshold=4), 5).startswith("fused_tb_kernel")
    assert P.kernel_name(P.DenoiseParams(border=P.BorderMode(1)), 5).startswith("fused_tb_kernel")


@pytest.mark.parametrize("w", [1, 2, 3, 31, 32, 33, 63, 64, 65, 481, 496, 511, 512, 513, 544, 1000, 1023, 1024,
                               1025, 1040, 1991, 1992, 1993, 2000, 2976, 3000, 3840])
def test_widths_across_layouts(w):
    _check(_sp(w, 57, w))


@pytest.mark.parametrize("h", [1, 2, 3, 4, 5, 9, 10, 11, 12, 13, 17, 36, 37, 45, 46, 47, 100, 321])
def test_heights_bands_and_tiles(h):
    _check(_sp(300, h, 7 * h))
    _check(_sp(700, h, 7 * h + 1))


@pytest.mark.parametrize("alpha", [1, 2, 19, 20, 64, 127, 128, 129, 200, 255])
def test_uniform_random_dense_candidates(alpha):
    rng = np.random.default_rng(alpha)
    _check(rng.integers(0, 256, (90, 1500), dtype=np.uint8), alpha=alpha)
    _check(rng.integers(0, 256, (70, 480), dtype=np.uint8), alpha=alpha)


def test_full_row_of_candidates():
    # alternating 0/255 columns: every interior pixel has no similar neighbour
    img = np.zeros((40, 1100), np.uint8)
    img[:, ::2] = 255
    img[::2] = 255 - img[::2]
    for thr in (1, 2, 3):
        _check(img, thr=thr)


@pytest.mark.parametrize("thr", [1, 2, 3])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 9, 12])
def test_iteration_chunks_and_thresholds(thr, k):
    _check(_sp(1500, 123, 100 * thr + k, 0.4), k=k, thr=thr)
    _check(_sp(481, 130, 100 * thr + k + 7, 0.6), k=k, thr=thr)


def test_batch_of_mixed_tiles():
    # an odd tile count: the last CTA's second tile is empty; neighbouring
    # tiles of one CTA belong to different images
    imgs = np.stack([_sp(481, 95, i, 0.1 + 0.1 * (i % 7)) for i in range(7)])
    out, stats = P.denoise_batch(imgs, P.DenoiseParams())
    for i in range(len(imgs)):
        ref_img, ref_stats = O.denoise(imgs[i])
        assert np.array_equal(out[i], ref_img), i
        assert [(s.flagged, s.replaced) for s in stats[i]] == ref_stats, i


def test_early_exit_converged_images():
    """The SURVEY KAT (constant 128 + 1% noise stops at iteration 3) at k=64:
    after the fixed point the launches only copy, so k=64 costs < 2x k=5
    (device time of the compute, phg_denoise's elapsed_ms)."""
    n = O.inject_sp_noise(np.full((321, 481), 128, np.uint8), 0.01, 0.5, 7)
    res = P.denoise(P.GrayImage.from_array(n), P.DenoiseParams(max_iterations=64))
    assert [s.replaced for s in res.stats] == [1526, 25, 0]
    big = O.inject_sp_noise(np.full((1400, 2000), 128, np.uint8), 0.01, 0.5, 7)
    g = P.GrayImage.from_array(big)

    def dev_ms(k):
        P.denoise(g, P.DenoiseParams(max_iterations=k))
        return min(P.denoise(g, P.DenoiseParams(max_iterations=k)).stats[0].elapsed_ms for _ in range(5))

    t5, t64 = dev_ms(5), dev_ms(64)
    assert t64 < 2.0 * t5, (t5, t64)
    ref_img, ref_stats = O.denoise(big, k=64)
    res = P.denoise(g, P.DenoiseParams(max_iterations=64))
    assert np.array_equal(res.image.pixels, ref_img)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats


def test_fp16_kernel_fallback_still_exact():
    """PHG_NO_BP=1 selects the round-1 fp16 two-tile kernel (kept as the A/B
    baseline); it must stay bit-exact."""
    code = ("import numpy as np, paper_1306_5390_b200 as P; from oracle import oracle as O;"
            "n=O.inject_sp_noise(O.synth_image(700,90,3),0.3,0.5,4);"
            "assert P.kernel_name(P.DenoiseParams(),5)=='fused_h2_kernel<T=5>';"
            "r=P.denoise(P.GrayImage.from_array(n),P.DenoiseParams());"
            "i,s=O.denoise(n); assert np.array_equal(r.image.pixels,i); "
            "assert [(x.flagged,x.replaced) for x in r.stats]==s; print('ok')")
    env = dict(os.environ, PHG_NO_BP="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("w", [1, 4, 33, 300, 511, 512, 513, 700, 1024, 1025, 1500, 1992, 1993])
def test_beta2_widths_across_layouts(w):
    """fused_bp2_kernel (beta = 2) over the three column layouts."""
    img = _sp(w, 41, 3 * w)
    res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(beta=2))
    ref_img, ref_stats = O.denoise(img, 20, 2)
    assert np.array_equal(res.image.pixels, ref_img), w
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, w


@pytest.mark.parametrize("h", [1, 2, 3, 4, 5, 6, 7, 9, 13, 17, 20, 21, 33, 45, 46, 100])
@pytest.mark.parametrize("k", [1, 4, 5])
def test_beta2_heights_bands(h, k):
    """Row counts around the beta = 2 band split (two steps per warp at least,
    the band-edge handover, the last warp's extra steps)."""
    img = _sp(600, h, 11 * h + k, 0.5)
    res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(beta=2, max_iterations=k))
    ref_img, ref_stats = O.denoise(img, 20, 2, k)
    assert np.array_equal(res.image.pixels, ref_img), (h, k)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, (h, k)


# ---- the single-buffer beta = 2 form (DIRECT: T = 1 launches of the resident
# path on wide regions store rows and replaced pixels straight to HBM; tiles
# of up to 90 staged rows, band-relative candidate items)

def _check2(img, alpha=20, k=5, thr=3):
    res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(alpha, 2, k, thr))
    ref_img, ref_stats = O.denoise(img, alpha, 2, k, thr, 0)
    assert np.array_equal(res.image.pixels, ref_img), (img.shape, alpha, k, thr)
    assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, (img.shape, alpha, k, thr)


@pytest.mark.parametrize("w,h", [(600, 86), (600, 87), (1025, 181), (2100, 300), (3000, 95), (1993, 173)])
@pytest.mark.parametrize("k", [1, 3])
def test_beta2_direct_tiles(w, h, k):
    """Row tiles around the 86-row output height, column tiles with aprons."""
    _check2(_sp(w, h, w + h + k, 0.5), k=k)


@pytest.mark.parametrize("alpha", [1, 30, 128, 129, 200])
def test_beta2_direct_dense_candidates(alpha):
    """Uniform-random pixels: whole rows of candidates in the band-relative
    list (rounds of 64, leftovers), both similarity forms (alpha <= 128 and
    > 128)."""
    rng = np.random.default_rng(alpha)
    _check2(rng.integers(0, 256, (190, 1500), dtype=np.uint8), alpha=alpha, k=2)


@pytest.mark.parametrize("thr", [1, 2, 3])
def test_beta2_direct_thresholds(thr):
    _check2(_sp(1100, 120, thr, 0.4), k=4, thr=thr)


def test_beta2_direct_early_exit():
    """A converged image (constant + 1% noise) at k = 64: after the fixed
    point the direct launches only copy the staged rows."""
    n = O.inject_sp_noise(np.full((200, 1500), 128, np.uint8), 0.01, 0.5, 9)
    _check2(n, k=64)


def test_beta2_direct_off_switch_same_result():
    """PHG_NO_DIRECT=1 keeps the two-buffer T = 1 form; both agree."""
    code = ("import numpy as np, paper_1306_5390_b200 as P; from oracle import oracle as O;"
            "n=O.inject_sp_noise(O.synth_image(1500,200,5),0.5,0.5,6);"
            "r=P.denoise(P.GrayImage.from_array(n),P.DenoiseParams(beta=2));"
            "i,s=O.denoise(n,20,2); assert np.array_equal(r.image.pixels,i); "
            "assert [(x.flagged,x.replaced) for x in r.stats]==s; print('ok')")
    env = dict(os.environ, PHG_NO_DIRECT="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("w,h", [(513, 90), (1025, 91), (1993, 181), (3000, 300), (1024, 7)])
@pytest.mark.parametrize("alpha", [20, 200])
def test_beta1_direct_single_iteration(w, h, alpha):
    """beta = 1, k = 1 on wide regions runs the single-buffer DIRECT form
    (92-row tiles, HBM stores from the sweep and the drain)."""
    _check(_sp(w, h, w * 7 + h, 0.4), alpha=alpha, k=1)


@pytest.mark.parametrize("n,w,beta,k", [(1, 31, 1, 5), (3, 481, 1, 5), (1, 300, 2, 5), (3, 200, 2, 1),
                                        (1, 100, 1, 1)])
def test_narrow_pairs_store_nothing_past_the_batch(n, w, beta, k):
    """Narrow tiles pair images (2p, 2p+1); with an odd batch the last CTA
    has no image 2p+1 and must not store anything for it.  A guard region
    after the batch in the same allocation stays untouched, and the stats
    (counters right behind it) stay exact."""
    import ctypes as C
    import torch
    from paper_1306_5390_b200._lib import PhgDevImage, check, lib
    h = 70
    pitch = (w + 15) // 16 * 16
    imgs = np.stack([_sp(w, h, 17 * i + w, 0.3) for i in range(n)])
    guard = 2 * h * pitch
    def dev(t):
        return PhgDevImage(t.data_ptr(), pitch, h * pitch, w, h, n, 0)
    bufs = []
    for fill in (0, 0xAB, 0xAB):
        t = torch.full((n * h * pitch + guard,), fill, dtype=torch.uint8, device="cuda")
        bufs.append(t)
    src = bufs[0][: n * h * pitch].view(n, h, pitch)
    src[:, :, :w] = torch.from_numpy(imgs).cuda()
    ctr = torch.zeros(2 * k * n + 64, dtype=torch.int64, device="cuda")
    ctr[2 * k * n:] = 0x5A5A
    params = P.DenoiseParams(20, beta, k, 3)._c()
    L = lib()
    s, d, t = dev(bufs[0]), dev(bufs[1]), dev(bufs[2])
    check(L.phg_dev_denoise(C.byref(s), C.byref(d), C.byref(t), C.byref(params), C.c_void_p(ctr.data_ptr()),
                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    for b in bufs[1:]:
        assert bool((b[n * h * pitch:] == 0xAB).all()), "store past the batch"
    assert bool((ctr[2 * k * n:] == 0x5A5A).all()), "counter store past the batch"
    out = bufs[1][: n * h * pitch].view(n, h, pitch)[:, :, :w].cpu().numpy()
    c = ctr[: 2 * k * n].view(n, k, 2).cpu().numpy()
    for i in range(n):
        ref_img, ref_stats = O.denoise(imgs[i], 20, beta, k)
        assert np.array_equal(out[i], ref_img), i
        got = [tuple(int(x) for x in c[i, j]) for j in range(len(ref_stats))]
        assert got == ref_stats, i


def test_random_shapes_and_plans():
    """Random widths (both layouts), heights, densities, alpha, thresholds and
    k (k = 1: the single-buffer DIRECT form on wide regions; k = 6, 7:
    two-launch plans) against the oracle, beta 1 and 2."""
    rng = np.random.default_rng(20261019)
    for _ in range(40):
        w, h = int(rng.integers(1, 2600)), int(rng.integers(1, 220))
        beta = int(rng.integers(1, 3))
        k = int(rng.choice([1, 2, 3, 6, 7]))
        thr = int(rng.integers(1, 4))
        alpha = int(rng.choice([5, 20, 60, 128, 129, 240]))
        img = _sp(w, h, int(rng.integers(0, 1 << 20)), float(rng.uniform(0.05, 0.7)))
        res = P.denoise(P.GrayImage.from_array(img), P.DenoiseParams(alpha, beta, k, thr))
        ref_img, ref_stats = O.denoise(img, alpha, beta, k, thr, 0)
        assert np.array_equal(res.image.pixels, ref_img), (w, h, beta, k, thr, alpha)
        assert [(s.flagged, s.replaced) for s in res.stats] == ref_stats, (w, h, beta, k, thr, alpha)
