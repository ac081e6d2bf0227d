"""SURVEY.md 8(f) rows f1/f4 around the denoise loop: the standalone
cardinality map (compute_cardinality, denoise.hpp:227-241) and its P2 dump
(`phgrms cardmap`, pgm.hpp:123-136), residual_noise_count
(metrics.hpp:52-59), and mse/psnr/format_db (metrics.hpp:18-50), on the
B200 through the C ABI, checked against the oracle and the reference's own
fixtures (test_cli.cpp:76-131, acceptance.cpp:305-320)."""
import math

import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

G = P.GrayImage


# ------------------------------------------------------------ host only
def test_write_p2_reference_fixtures():
    assert P.write_p2(3, 3, O.cardinality(np.full((3, 3), 100, np.uint8), 20, 1).reshape(-1), 9) == \
        "P2\n3 3\n9\n4 6 4\n6 9 6\n4 6 4\n"
    imp = np.full((3, 3), 100, np.uint8)
    imp[1, 1] = 255
    assert P.write_p2(3, 3, O.cardinality(imp, 20, 1).reshape(-1), 9) == "P2\n3 3\n9\n3 5 3\n5 1 5\n3 5 3\n"
    assert P.write_p2(2, 1, [0, 1000], 65535) == "P2\n2 1\n65535\n0 1000\n"


def test_format_db_rendering():
    assert P.format_db(P.PsnrValue(math.inf)) == "inf"
    assert P.format_db(P.PsnrValue(24.04799)) == "24.048"
    assert P.format_db(P.PsnrValue(0.0)) == "0.000"


# ------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_psnr_reference_fixtures():
    a = G(8, 8, 40)
    b = G.from_array(np.full((8, 8), 56, np.uint8))
    assert P.mse(a, a) == 0.0 and P.psnr(a, a).infinite() and P.format_db(P.psnr(a, a)) == "inf"
    assert P.mse(a, b) == 256.0 and P.format_db(P.psnr(a, b)) == "24.048"
    assert P.format_db(P.psnr(G(1, 1, 0), G(1, 1, 255))) == "0.000"
    with pytest.raises(P.InvalidArgument, match="mse: image dimensions differ"):
        P.mse(G(4, 4, 1), G(4, 5, 1))


@pytest.mark.gpu
@pytest.mark.parametrize("w,h", [(1, 1), (15, 3), (16, 16), (17, 9), (481, 321), (3840, 2160), (4097, 1000)])
def test_mse_exact(w, h):
    rng = np.random.default_rng(w * 131 + h)
    x = rng.integers(0, 256, (h, w), dtype=np.uint8)
    y = rng.integers(0, 256, (h, w), dtype=np.uint8)
    ref = int(((x.astype(np.int64) - y) ** 2).sum())
    assert P.mse(G.from_array(x), G.from_array(y)) == ref / (w * h)
    z = np.full((h, w), 255, np.uint8)
    zz = np.zeros((h, w), np.uint8)
    assert P.mse(G.from_array(z), G.from_array(zz)) == 65025.0


@pytest.mark.gpu
def test_residual_noise_count_vs_oracle():
    rng = np.random.default_rng(55)
    for _ in range(60):
        w, h = int(rng.integers(1, 1100)), int(rng.integers(1, 90))
        alpha, beta = int(rng.integers(1, 256)), int(rng.integers(1, 4))
        thr = int(rng.choice([1, 2, 3, 4, 9, 26, 1000, 5000]))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        ref = int(np.count_nonzero(O.cardinality(img, alpha, beta) < thr))
        assert P.residual_noise_count(G.from_array(img), alpha, beta, thr) == ref, (w, h, alpha, beta, thr)


@pytest.mark.gpu
def test_residual_noise_count_denoised_bsds():
    clean = O.synth_image(481, 321, 1)
    noisy = O.inject_sp_noise(clean, 0.10, 0.5, 12345)
    den, _ = O.denoise(noisy)
    for img in (noisy, den):
        ref = int(np.count_nonzero(O.cardinality(img, 20, 1) < 3))
        assert P.residual_noise_count(G.from_array(img), 20, 1, 3) == ref


@pytest.mark.gpu
def test_cardinality_map_fast_path_vs_oracle():
    rng = np.random.default_rng(77)
    for _ in range(40):
        w, h = int(rng.integers(1, 1500)), int(rng.integers(1, 120))
        alpha = int(rng.integers(1, 256))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = P.compute_cardinality(G.from_array(img), alpha, 1).counts.reshape(h, w)
        assert np.array_equal(got, O.cardinality(img, alpha, 1)), (w, h, alpha)


@pytest.mark.gpu
def test_cardmap_p2_on_gpu():
    assert P.cardmap(G(3, 3, 100)) == "P2\n3 3\n9\n4 6 4\n6 9 6\n4 6 4\n"
    imp = G(3, 3, 100)
    imp.set(1, 1, 255)
    assert P.cardmap(imp) == "P2\n3 3\n9\n3 5 3\n5 1 5\n3 5 3\n"
    assert P.cardmap(G(3, 3, 100), beta=2)[:9] == "P2\n3 3\n25"


@pytest.mark.gpu
@pytest.mark.parametrize("beta", [1, 2])
@pytest.mark.parametrize("alpha", [1, 20, 200])
@pytest.mark.parametrize("border", [0, 1])
def test_denoise_pass_tiled_vs_oracle(beta, alpha, border):
    # denoise_pass with a caller-supplied map (denoise.hpp:243-283) on the
    # tiled kernel: multi-tile shapes, the true map and arbitrary maps
    rng = np.random.default_rng(alpha * 7 + border + 100 * beta)
    for w, h in ((700, 301), (257, 17), (1023, 64), (5, 3)):
        img = O.inject_sp_noise(O.synth_image(w, h, w + h), 0.3, 0.5, alpha)
        for kind in ("true", "random"):
            card = O.cardinality(img, alpha, beta) if kind == "true" else \
                rng.integers(0, 26, (h, w)).astype(np.int32)
            for thr in (1, 3, 7, 30):
                p = P.DenoiseParams(alpha, beta, 1, thr, P.BorderMode(border))
                out, st = P.denoise_pass(G.from_array(img), P.CardinalityMap(w, h, card.reshape(-1)), p)
                ref, f, r = O.removal_pass(img, card, alpha, beta, thr, border)
                assert np.array_equal(out.pixels, ref), (w, h, kind, thr)
                assert (st.flagged, st.replaced) == (f, r)


@pytest.mark.gpu
def test_cardinality_map_beta2_staged_vs_oracle():
    # compute_cardinality with beta = 2 runs the byte-SIMD kernel in CARD mode
    rng = np.random.default_rng(91)
    for w, h in ((1, 1), (3, 70), (497, 33), (1100, 130), (2000, 67)):
        alpha = int(rng.integers(1, 256))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        got = P.compute_cardinality(G.from_array(img), alpha, 2).counts.reshape(h, w)
        assert np.array_equal(got, O.cardinality(img, alpha, 2)), (w, h, alpha)
    assert P.cardmap(G(3, 3, 100), beta=2) == "P2\n3 3\n25\n9 12 9\n12 16 12\n9 12 9\n" or \
        P.cardmap(G(3, 3, 100), beta=2)[:9] == "P2\n3 3\n25"


@pytest.mark.gpu
@pytest.mark.parametrize("n,w,h", [(1, 481, 321), (3, 481, 321), (2, 300, 95), (1, 1500, 400), (2, 2100, 181),
                                   (3, 17, 200), (1, 1024, 1)])
@pytest.mark.parametrize("thr,alpha", [(3, 20), (2, 20), (1, 20), (3, 200)])
def test_residual_count_packed_bit_batches(n, w, h, thr, alpha):
    """beta = 1, card_threshold <= 3 runs the packed-bit sweep's count-only
    form (fused_bp_kernel COUNT, up to 92-row tiles, both column layouts):
    per-image counts of C < thr over batches, against the oracle's map."""
    import ctypes as C
    import torch
    from paper_1306_5390_b200._lib import PhgDevImage, check, lib
    pitch = (w + 15) // 16 * 16
    imgs = np.stack([O.inject_sp_noise(O.synth_image(w, h, 5 * i + w), 0.1 + 0.2 * i, 0.5, i + 1)
                     for i in range(n)])
    buf = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")
    buf[:, :, :w] = torch.from_numpy(imgs).cuda()
    counts = torch.zeros(n + 4, dtype=torch.int64, device="cuda")
    im = PhgDevImage(buf.data_ptr(), pitch, h * pitch, w, h, n, 0)
    check(lib().phg_dev_residual_count(C.byref(im), alpha, 1, thr, C.c_void_p(counts.data_ptr()),
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    got = counts.cpu().numpy()
    for i in range(n):
        ref = int(np.count_nonzero(O.cardinality(imgs[i], alpha, 1) < thr))
        assert int(got[i]) == ref, (i, n, w, h, thr, alpha)
    assert not got[n:].any()
