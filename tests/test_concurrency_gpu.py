"""Concurrent callers (SPEC.md:77 -- the reference's functions are pure and
"safe to call from any number of concurrent callers").  Every calling thread
gets its own streams and scratch buffers per device, so calls from several
host threads on one device overlap and stay bit-exact against the oracle.
ctypes releases the GIL for the duration of each C call."""
import threading

import numpy as np
import pytest

import paper_1306_5390_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run_threads(fns):
    errors = []

    def wrap(fn):
        try:
            fn()
        except BaseException as e:  # noqa: BLE001 -- reported below
            errors.append(e)

    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errors:
        raise errors[0]


def test_concurrent_denoise_calls_on_one_device():
    cases = []
    for i in range(8):
        w, h = [(481, 321), (640, 480), (1000, 77), (3840, 2160)][i % 4]
        beta = 1 + (i % 3 == 2)
        img = O.inject_sp_noise(O.synth_image(w, h, 50 + i), 0.1 + 0.08 * i, 0.5, i)
        cases.append((img, P.DenoiseParams(20, beta, 5 + i % 2, 3)))
    refs = [O.denoise(img, p.alpha, p.beta, p.max_iterations, p.card_threshold, 0) for img, p in cases]
    results = [None] * len(cases)

    def job(i):
        def f():
            for _ in range(3):  # repeated calls reuse the thread's buffers
                img, p = cases[i]
                r = P.denoise(P.GrayImage.from_array(img), p)
                results[i] = (r.image.pixels.copy(), [(s.flagged, s.replaced) for s in r.stats])
        return f

    _run_threads([job(i) for i in range(len(cases))])
    for (out, st), (ref, ref_st) in zip(results, refs):
        assert np.array_equal(out, ref)
        assert st == ref_st


def test_concurrent_mixed_entry_points():
    img = O.inject_sp_noise(O.synth_image(700, 300, 9), 0.3, 0.5, 4)
    g = P.GrayImage.from_array(img)
    ref_img, ref_st = O.denoise(img)
    ref_card = O.cardinality(img, 20, 2)
    batch = np.stack([img, img[::-1].copy()])
    ref_b1, _ = O.denoise(batch[1])
    out = {}

    def a():
        for _ in range(4):
            out["d"] = P.denoise(g, P.DenoiseParams()).image.pixels.copy()

    def b():
        for _ in range(4):
            out["c"] = np.asarray(P.compute_cardinality(g, 20, 2).counts).reshape(img.shape).copy()

    def c():
        for _ in range(4):
            out["b"] = P.denoise_batch(batch, P.DenoiseParams())[0].copy()

    def d():
        for _ in range(4):
            out["r"] = P.residual_noise_count(g, 20, 2, 3)

    _run_threads([a, b, c, d])
    assert np.array_equal(out["d"], ref_img)
    assert np.array_equal(out["c"], ref_card.reshape(img.shape))
    assert np.array_equal(out["b"][0], ref_img) and np.array_equal(out["b"][1], ref_b1)
    assert out["r"] == int((ref_card < 3).sum())
