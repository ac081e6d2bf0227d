"""ctypes loader for the parity CHECKER (test infrastructure only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_1306_5390_b200``) never does.

Two libraries:
  * ``liboracle.so``           -- plain-C restatement (oracle/phgrms_oracle.c)
  * ``_ref/libphgrms_ref.so``  -- the reference's own headers compiled in place
                                  (oracle/ref_shim.cpp); absent if the reference
                                  tree was never available when building.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


class _Params(C.Structure):
    _fields_ = [("alpha", C.c_int), ("beta", C.c_int), ("max_iterations", C.c_int),
                ("card_threshold", C.c_int), ("border", C.c_int)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_LIB = None
_REF = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.orc_synth_image.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_int, _u8p]
        L.orc_inject_sp_noise.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_uint32, _u8p, C.c_void_p]
        L.orc_inject_sp_noise.restype = C.c_longlong
        L.orc_cardinality.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.orc_cardinality_scatter.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.orc_rms_replacement.argtypes = [C.c_uint64, C.c_int]
        L.orc_removal_pass.argtypes = [_u8p, _i32p, C.c_int, C.c_int, C.POINTER(_Params), _u8p,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.orc_denoise.argtypes = [_u8p, C.c_int, C.c_int, C.POINTER(_Params), _u8p, _i64p, _i64p,
                                  C.POINTER(C.c_int)]
        L.orc_row_blocks.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_band_pass.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.POINTER(_Params), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64)]
        L.orc_mt19937_nth.argtypes = [C.c_uint32, C.c_uint64]
        L.orc_mt19937_nth.restype = C.c_uint32
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libphgrms_ref.so"))


def ref():
    """The reference itself (compiled from /root/reference headers)."""
    global _REF
    if _REF is None:
        R = C.CDLL(os.path.join(HERE, "_ref", "libphgrms_ref.so"))
        R.ref_synth_image.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_int, _u8p]
        R.ref_inject_sp_noise.argtypes = [_u8p, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_uint32, _u8p, C.c_void_p]
        R.ref_inject_sp_noise.restype = C.c_longlong
        R.ref_compute_cardinality.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        R.ref_cardinality_scatter.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        R.ref_denoise_pass.argtypes = [_u8p, _i32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, _u8p, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]
        R.ref_oracle_removal_pass.argtypes = [_u8p, _i32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_int, C.c_int, _u8p]
        R.ref_denoise.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, _u8p, _i64p, _i64p, C.POINTER(C.c_int)]
        R.ref_denoise_batch.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_int, _u8p, _i32p]
        R.ref_denoise_batch_stats.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.c_int, _u8p, _i64p, _i64p, _i32p]
        R.ref_denoise_band.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, C.c_int, _u8p, _i64p, _i64p]
        R.ref_hardware_concurrency.restype = C.c_int
        _REF = R
    return _REF


# ---------------------------------------------------------------- helpers
def synth_image(w, h, seed, kind=2):
    out = np.empty((h, w), np.uint8)
    assert lib().orc_synth_image(w, h, seed, kind, out) == 0
    return out


def inject_sp_noise(img, density, salt_ratio=0.5, seed=0, with_mask=False):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    mask = np.empty_like(img) if with_mask else None
    n = lib().orc_inject_sp_noise(img, w, h, density, salt_ratio, seed, out,
                                  mask.ctypes.data if with_mask else None)
    assert n >= 0
    return (out, mask) if with_mask else out


def cardinality(img, alpha, beta):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty((h, w), np.int32)
    assert lib().orc_cardinality(img, w, h, alpha, beta, out) == 0
    return out


def cardinality_scatter(img, alpha, beta):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty((h, w), np.int32)
    lib().orc_cardinality_scatter(img, w, h, alpha, beta, out)
    return out


def rms_replacement(sum_sq, flag):
    return lib().orc_rms_replacement(sum_sq, flag)


def _params(alpha=20, beta=1, k=5, thr=3, border=0):
    return _Params(alpha, beta, k, thr, border)


def removal_pass(img, card, alpha=20, beta=1, thr=3, border=0):
    img = np.ascontiguousarray(img, np.uint8)
    card = np.ascontiguousarray(card, np.int32)
    h, w = img.shape
    out = np.empty_like(img)
    f, r = C.c_int64(), C.c_int64()
    p = _params(alpha, beta, 1, thr, border)
    assert lib().orc_removal_pass(img, card, w, h, C.byref(p), out, C.byref(f), C.byref(r)) == 0
    return out, f.value, r.value


def denoise(img, alpha=20, beta=1, k=5, thr=3, border=0):
    """Returns (image, [(flagged, replaced), ...]) -- one entry per executed
    iteration, exactly like phgrms::denoise (denoise.hpp:292-311)."""
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    fl = np.zeros(k, np.int64)
    rp = np.zeros(k, np.int64)
    it = C.c_int()
    p = _params(alpha, beta, k, thr, border)
    assert lib().orc_denoise(img, w, h, C.byref(p), out, fl, rp, C.byref(it)) == 0
    return out, [(int(fl[i]), int(rp[i])) for i in range(it.value)]


def band_pass(src, dst, row_base, height, y_lo, y_hi, c_lo, c_hi, alpha=20, beta=1, thr=3, border=0):
    """One iteration on a band buffer (see orc_band_pass); returns (flagged, replaced)."""
    rows, w = src.shape
    f, r = C.c_int64(), C.c_int64()
    p = _params(alpha, beta, 1, thr, border)
    rc = lib().orc_band_pass(src, dst, w, rows, row_base, height, y_lo, y_hi, c_lo, c_hi, C.byref(p),
                             C.byref(f), C.byref(r))
    if rc != 0:
        raise ValueError(f"band_pass: band does not hold the rows it needs (rc={rc})")
    return f.value, r.value


def row_blocks(height, workers):
    b = (C.c_int * max(workers, 1))()
    e = (C.c_int * max(workers, 1))()
    n = lib().orc_row_blocks(height, workers, b, e)
    if n < 0:
        raise ValueError("row_blocks: bad height or worker count")
    return [(b[i], e[i]) for i in range(n)]


# ------------------------------------------------- the reference itself
def ref_denoise(img, alpha=20, beta=1, k=5, thr=3, border=0, workers=1):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    fl = np.zeros(k, np.int64)
    rp = np.zeros(k, np.int64)
    it = C.c_int()
    assert ref().ref_denoise(img, w, h, alpha, beta, k, thr, border, workers, out, fl, rp,
                             C.byref(it)) == 0
    return out, [(int(fl[i]), int(rp[i])) for i in range(it.value)]


def ref_cardinality(img, alpha, beta, workers=1):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty((h, w), np.int32)
    assert ref().ref_compute_cardinality(img, w, h, alpha, beta, workers, out) == 0
    return out


def ref_synth_image(w, h, seed, kind=2):
    out = np.empty((h, w), np.uint8)
    assert ref().ref_synth_image(w, h, seed, kind, out) == 0
    return out


def ref_inject_sp_noise(img, density, salt_ratio=0.5, seed=0, with_mask=False):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    mask = np.empty_like(img) if with_mask else None
    n = ref().ref_inject_sp_noise(img, w, h, density, salt_ratio, seed, out,
                                  mask.ctypes.data if with_mask else None)
    assert n >= 0
    return (out, mask) if with_mask else out


def ref_denoise_batch(imgs, alpha=20, beta=1, k=5, thr=3, border=0, threads=1):
    imgs = np.ascontiguousarray(imgs, np.uint8)
    n, h, w = imgs.shape
    out = np.empty_like(imgs)
    its = np.zeros(n, np.int32)
    ref().ref_denoise_batch(imgs, n, w, h, alpha, beta, k, thr, border, threads, out, its)
    return out, its


def ref_denoise_batch_stats(imgs, alpha=20, beta=1, k=5, thr=3, border=0, threads=1):
    """The reference on a packed batch: (final images, per-image stats lists)."""
    imgs = np.ascontiguousarray(imgs, np.uint8)
    n, h, w = imgs.shape
    out = np.empty_like(imgs)
    fl = np.zeros((n, k), np.int64)
    rp = np.zeros((n, k), np.int64)
    its = np.zeros(n, np.int32)
    assert ref().ref_denoise_batch_stats(imgs, n, w, h, alpha, beta, k, thr, border, threads, out, fl, rp,
                                         its) == 0
    return out, [[(int(fl[i, j]), int(rp[i, j])) for j in range(its[i])] for i in range(n)]


def ref_denoise_band(band, own_lo, own_hi, alpha=20, beta=1, k=5, thr=3, border=0):
    """k reference passes on a row band; (owned rows after k passes, owned
    per-pass (flagged, replaced) over all k passes, untruncated)."""
    band = np.ascontiguousarray(band, np.uint8)
    bh, w = band.shape
    out = np.empty((own_hi - own_lo, w), np.uint8)
    fl = np.zeros(k, np.int64)
    rp = np.zeros(k, np.int64)
    assert ref().ref_denoise_band(band, w, bh, own_lo, own_hi, alpha, beta, k, thr, border, out, fl, rp) == 0
    return out, [(int(fl[i]), int(rp[i])) for i in range(k)]


# ---------------------------------------------------------------------------
# The on-device counter-based generators (kernel_gen.cuh)
# restated in numpy.  These are NEW generators (not the reference's mt19937
# streams); this restatement is their parity checker.
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _gen_index(n, h, w):
    img = np.arange(n, dtype=np.uint64)[:, None, None]
    r = np.arange(h, dtype=np.uint64)[None, :, None]
    c = np.arange(w, dtype=np.uint64)[None, None, :]
    with np.errstate(over="ignore"):
        return (img * np.uint64(h) + r) * np.uint64(w) + c


def dev_smooth(w, h, seed, n=1):
    """phg_dev_synth_smooth: field = mix64(seed*K + index) & 0xff, then the
    clamped 3x3 mean with round-half-up (image.hpp:87-101 smoothing)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * np.uint64(0xD1342543DE82EF95)
        field = (_mix64(base + _gen_index(n, h, w)) & np.uint64(0xFF)).astype(np.int64)
    pad = np.pad(field, ((0, 0), (1, 1), (1, 1)))
    ones = np.pad(np.ones((n, h, w), np.int64), ((0, 0), (1, 1), (1, 1)))
    s = sum(pad[:, 1 + dy:1 + dy + h, 1 + dx:1 + dx + w] for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    cnt = sum(ones[:, 1 + dy:1 + dy + h, 1 + dx:1 + dx + w] for dy in (-1, 0, 1) for dx in (-1, 0, 1))
    return ((s + cnt // 2) // cnt).astype(np.uint8)


def dev_noise(imgs, density, salt_ratio, seed):
    """phg_dev_inject_noise: Bernoulli(density) per pixel from
    mix64(seed*K + index), salt iff mix64(draw) < salt_ratio * 2^64."""
    imgs = np.array(imgs, dtype=np.uint8, copy=True)
    if imgs.ndim == 2:
        imgs = imgs[None]
    n, h, w = imgs.shape
    if density == 0.0:
        return imgs, 0
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * np.uint64(0xD1342543DE82EF95)
        u = _mix64(base + _gen_index(n, h, w))
    hit = np.ones_like(u, dtype=bool) if density >= 1.0 else u < np.uint64(int(math.ldexp(density, 64)))
    if salt_ratio >= 1.0:
        salt = np.ones_like(hit)
    else:
        salt = _mix64(u) < np.uint64(int(math.ldexp(salt_ratio, 64)))
    imgs[hit] = np.where(salt[hit], 255, 0).astype(np.uint8)
    return imgs, int(hit.sum())
