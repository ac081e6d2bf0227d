"""the on-device counter-based generators
(kernel_gen.cuh) against their numpy restatement (oracle.dev_smooth /
dev_noise), plus the properties that make them usable for giga-pixel inputs:
determinism, Bernoulli statistics, and no 2^32-pixel limit."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O


def test_restatement_statistics_cpu():
    img = O.dev_smooth(640, 480, 5)
    assert img.min() >= 0 and 60 < img.mean() < 195  # a 3x3 mean of uniform bytes
    noisy, cnt = O.dev_noise(img, 0.3, 0.5, 11)
    n = img.size
    assert abs(cnt - 0.3 * n) < 6 * np.sqrt(n * 0.3 * 0.7)
    salt = int((noisy[0] == 255).sum() - (img == 255).sum())
    assert abs(salt - 0.5 * cnt) < 6 * np.sqrt(cnt * 0.25) + (img == 255).sum()
    again, cnt2 = O.dev_noise(img, 0.3, 0.5, 11)
    assert cnt2 == cnt and np.array_equal(again, noisy)
    assert O.dev_noise(img, 0.0, 0.5, 1)[1] == 0 and O.dev_noise(img, 1.0, 1.0, 1)[0].min() == 255


@pytest.mark.gpu
@pytest.mark.parametrize("n,w,h,seed", [(1, 1, 1, 0), (1, 7, 5, 3), (3, 481, 321, 1), (2, 1000, 37, 2**40 + 7)])
def test_device_generators_match_restatement(n, w, h, seed):
    import torch

    from paper_1306_5390_b200._lib import PhgDevImage, check, lib

    L = lib()
    pitch = (w + 15) // 16 * 16
    t = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")
    check(L.phg_dev_synth_smooth(C.byref(_im(PhgDevImage, t, w, h, n)), 0, h, seed, None))
    torch.cuda.synchronize()
    clean = O.dev_smooth(w, h, seed, n)
    assert np.array_equal(t[:, :, :w].cpu().numpy(), clean)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for density, salt in ((0.3, 0.5), (0.05, 0.0), (1.0, 1.0), (0.7, 0.25)):
        t2 = t.clone()
        cnt.zero_()
        check(L.phg_dev_inject_noise(C.byref(_im(PhgDevImage, t2, w, h, n)), 0, h, density, salt, seed ^ 5,
                                     C.c_void_p(cnt.data_ptr()), None))
        torch.cuda.synchronize()
        ref, rc = O.dev_noise(clean, density, salt, seed ^ 5)
        assert np.array_equal(t2[:, :, :w].cpu().numpy(), ref), (density, salt)
        assert int(cnt.item()) == rc


def _im(cls, t, w, h, n):
    im = cls()
    im.data, im.pitch, im.image_stride = t.data_ptr(), t.shape[-1], t.shape[-1] * h
    im.width, im.rows, im.n_images = w, h, n
    return im


@pytest.mark.gpu
def test_beyond_2_32_pixels():
    # the reference injector divides by zero at 2^32 pixels;
    # the counter-based one covers a 65536 x 65537 image in one call
    import torch

    from paper_1306_5390_b200._lib import PhgDevImage, check, lib

    L = lib()
    w, h = 65536, 65537
    t = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    im = _im(PhgDevImage, t[None], w, h, 1)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    check(L.phg_dev_synth_smooth(C.byref(im), 0, h, 1, None))
    check(L.phg_dev_inject_noise(C.byref(im), 0, h, 0.3, 0.5, 12345, C.c_void_p(cnt.data_ptr()), None))
    torch.cuda.synchronize()
    n = w * h
    assert abs(int(cnt.item()) - 0.3 * n) < 6 * (n * 0.21) ** 0.5
    # spot-check the last rows (counter indices above 2^32) against the
    # restatement evaluated on that block only
    tail = t[h - 3:, :64].cpu().numpy()
    assert np.array_equal(tail, _block(w, h, 1, 12345, 0.3, 0.5, h - 3, h, 0, 64))
    del t


def _block(w, h, seed, nseed, density, salt, r0, r1, c0, c1):
    """oracle.dev_smooth + dev_noise for rows [r0, r1) x cols [c0, c1) of a
    single w x h image, without materialising the whole image."""
    K = np.uint64(0xD1342543DE82EF95)
    rr = np.arange(max(0, r0 - 1), min(h, r1 + 1), dtype=np.uint64)
    cc = np.arange(max(0, c0 - 1), min(w, c1 + 1), dtype=np.uint64)
    with np.errstate(over="ignore"):
        idx = rr[:, None] * np.uint64(w) + cc[None, :]
        field = (O._mix64(np.uint64(seed) * K + idx) & np.uint64(0xFF)).astype(np.int64)
    out = np.empty((r1 - r0, c1 - c0), np.uint8)
    for i, r in enumerate(range(r0, r1)):
        for j, c in enumerate(range(c0, c1)):
            ys = [y for y in (r - 1, r, r + 1) if 0 <= y < h]
            xs = [x for x in (c - 1, c, c + 1) if 0 <= x < w]
            vals = [field[y - int(rr[0]), x - int(cc[0])] for y in ys for x in xs]
            out[i, j] = (sum(vals) + len(vals) // 2) // len(vals)
    with np.errstate(over="ignore"):
        ridx = np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(w) + np.arange(c0, c1, dtype=np.uint64)[None, :]
        u = O._mix64(np.uint64(nseed) * K + ridx)
    hit = u < np.uint64(int(np.ldexp(density, 64)))
    is_salt = O._mix64(u) < np.uint64(int(np.ldexp(salt, 64)))
    out[hit] = np.where(is_salt[hit], 255, 0)
    return out


@pytest.mark.gpu
def test_row_band_generation_equals_whole_image():
    # a band generated with row_base/height equals the same rows of the image
    import torch

    from paper_1306_5390_b200._lib import PhgDevImage, check, lib

    L = lib()
    w, h = 300, 97
    pitch = 304
    full = torch.zeros((1, h, pitch), dtype=torch.uint8, device="cuda")
    check(L.phg_dev_synth_smooth(C.byref(_im(PhgDevImage, full, w, h, 1)), 0, h, 42, None))
    check(L.phg_dev_inject_noise(C.byref(_im(PhgDevImage, full, w, h, 1)), 0, h, 0.4, 0.5, 7, None, None))
    for lo, hi in ((0, 30), (30, 61), (61, 97)):
        band = torch.zeros((1, hi - lo, pitch), dtype=torch.uint8, device="cuda")
        check(L.phg_dev_synth_smooth(C.byref(_im(PhgDevImage, band, w, hi - lo, 1)), lo, h, 42, None))
        check(L.phg_dev_inject_noise(C.byref(_im(PhgDevImage, band, w, hi - lo, 1)), lo, h, 0.4, 0.5, 7, None, None))
        torch.cuda.synchronize()
        assert torch.equal(band[0, :, :w], full[0, lo:hi, :w])
