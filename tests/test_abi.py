"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/phgrms_b200.h declares, and its host-only entry points (parameter
validation, stats finalisation, input generators) behave like the reference.
No compute call is made here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1306_5390_b200 as P
from paper_1306_5390_b200._lib import EXPORTS, PhgParams, PhgPassStats, lib
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "phgrms_b200.h")).read()
    return sorted(set(re.findall(r"\b(phg_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    L = lib()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(EXPORTS)
    assert L.phg_abi_version() == 1


def test_validation_messages_match_reference():
    L = lib()
    cases = [((0, 1, 5, 3, 0), "alpha must be in [1, 255]"), ((256, 1, 5, 3, 0), "alpha must be in [1, 255]"),
             ((20, 0, 5, 3, 0), "beta must be >= 1"), ((20, 1, 0, 3, 0), "iterations must be >= 1"),
             ((20, 1, 5, 0, 0), "card_threshold must be >= 1")]
    for args, msg in cases:
        assert L.phg_validate_params(C.byref(PhgParams(*args))) == -1
        assert L.phg_last_error().decode() == msg
    assert L.phg_validate_params(C.byref(PhgParams(20, 1, 5, 3, 0))) == 0
    with pytest.raises(P.InvalidArgument, match="beta must be >= 1"):
        P.DenoiseParams(beta=0).validate()


def test_python_mirror_defaults_and_helpers():
    p = P.DenoiseParams()
    assert (p.alpha, p.beta, p.max_iterations, p.card_threshold, p.border) == (20, 1, 5, 3, P.BorderMode.Faithful)
    assert P.similar(100, 119, 20) and P.similar(119, 100, 20)
    assert not P.similar(100, 120, 20) and not P.similar(10, 11, 1)
    assert [(b.begin, b.end) for b in P.row_blocks(1000, 3)] == O.row_blocks(1000, 3)
    assert len(P.row_blocks(5, 8)) == 5
    with pytest.raises(P.InvalidArgument):
        P.row_blocks(-1, 2)
    with pytest.raises(P.InvalidArgument, match="image dimensions must be >= 1"):
        P.GrayImage(0, 3)
    visits = [0] * 37
    P.parallel_for_rows(37, 5, lambda lo, hi: [visits.__setitem__(r, visits[r] + 1) for r in range(lo, hi)])
    assert visits == [1] * 37
    with pytest.raises(RuntimeError, match="boom"):
        P.parallel_for_rows(8, 4, lambda lo, hi: (_ for _ in ()).throw(RuntimeError("boom")) if lo == 0 else None)


def test_rms_replacement_integer_rule_matches_reference_double():
    # exhaustive over beta=1 windows (f <= 8) on a strided S range + all ties
    for f in range(1, 9):
        for S in list(range(0, 2000)) + list(range(0, f * 65025 + 1, 97)):
            assert P.rms_replacement(S, f) == O.rms_replacement(S, f), (S, f)
        for u in range(1, 256):  # exact .5 ties: 4S = (2u-1)^2 f
            if ((2 * u - 1) ** 2 * f) % 4 == 0:
                S = (2 * u - 1) ** 2 * f // 4
                assert P.rms_replacement(S, f) == O.rms_replacement(S, f) == u


def test_finalize_stats_truncates_after_first_zero_replacement():
    L = lib()
    ctr = np.array([[[9, 5], [4, 0], [4, 0]], [[3, 3], [2, 2], [1, 1]]], np.uint64)
    stats = (PhgPassStats * 6)()
    its = (C.c_int * 2)()
    assert L.phg_finalize_stats(ctr.ctypes.data, 2, 3, stats, its) == 0
    assert list(its) == [2, 3]
    assert [(s.iteration, s.flagged, s.replaced) for s in stats[:2]] == [(1, 9, 5), (2, 4, 0)]
    assert [(s.iteration, s.replaced) for s in stats[3:6]] == [(1, 3), (2, 2), (3, 1)]


def test_host_generators_match_oracle():
    for seed in (0, 1, 77, 2**31 + 5):
        for kind in (0, 1, 2):
            a = P.synth_image(53, 29, seed, P.SynthKind(kind))
            assert np.array_equal(a.pixels, O.synth_image(53, 29, seed & 0xFFFFFFFF, kind))
        for d in (0.0, 0.05, 0.5, 1.0):
            noisy, mask = P.inject_sp_noise(a, P.NoiseSpec(d, 0.4, seed), with_mask=True)
            on, om = O.inject_sp_noise(a.pixels, d, 0.4, seed & 0xFFFFFFFF, with_mask=True)
            assert np.array_equal(noisy.pixels, on) and np.array_equal(mask, om)
    with pytest.raises(P.InvalidArgument, match="density must be in"):
        P.inject_sp_noise(P.GrayImage(3, 3), P.NoiseSpec(1.5))


def test_workload_generator_matches_reference_digest():
    import hashlib
    import json
    from paper_1306_5390_b200 import workloads as WL
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
    for e in d["c4_first16"][:4]:
        assert hashlib.sha256(WL.c4_image(e["i"]).tobytes()).hexdigest() == e["noisy"]
    assert hashlib.sha256(WL.single_image("c1").tobytes()).hexdigest() == d["c1"]["noisy"]


def test_compute_entry_points_fail_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(P.CudaError):
        P.compute_cardinality(P.GrayImage(4, 4, 1), 20, 1)


def test_sharded_argument_errors_without_gpu():
    # phg_denoise_sharded validates the parameters and the device list
    # before touching CUDA; with no GPU the device check fails loudly
    img = np.zeros((4, 4), np.uint8)
    with pytest.raises(P.InvalidArgument, match="alpha must be in"):
        P.denoise_sharded(img, P.DenoiseParams(alpha=0), [0])
    with pytest.raises(P.InvalidArgument, match="devices must list at least one GPU"):
        P.denoise_sharded(img, P.DenoiseParams(), [])
    try:
        import torch
        if torch.cuda.is_available():
            return
    except ImportError:
        pass
    with pytest.raises(P.CudaError):
        P.denoise_sharded(img, P.DenoiseParams(), [0])


def test_launch_plan_host_only():
    """phg_launch_plan is host logic (no device needed): the resident path's
    launches per parameter set and image size."""
    L = lib()

    def plan(args, w, h, n, cap=64):
        buf = (C.c_int * cap)()
        k = L.phg_launch_plan(C.byref(PhgParams(*args)), w, h, n, buf, cap)
        return list(buf[:k]) if k >= 0 else k

    assert plan((20, 1, 5, 3, 0), 481, 321, 4096) == [5]          # C4: one T=5 launch
    assert plan((20, 1, 5, 3, 0), 3840, 2160, 1) == [5]           # C2
    assert plan((20, 1, 5, 3, 0), 65536, 65536, 1) == [1] * 5     # C5: single-buffer T=1 launches
    assert plan((20, 1, 12, 3, 0), 481, 321, 1) == [4, 4, 4]
    assert plan((20, 2, 5, 3, 0), 16384, 16384, 1) == [1] * 5     # C3
    assert plan((20, 1, 5, 3, 1), 4000, 4000, 1) == [5]           # InBounds: fused_tb_kernel
    assert plan((20, 4, 3, 3, 0), 100, 100, 1) == [1, 1, 1]       # beta >= 4: scalar kernel
    assert plan((20, 1, 5, 3, 0), 0, 10, 1) < 0
    assert plan((20, 1, 5, 3, 0), 481, 321, 1, cap=0) < 0
    assert L.phg_launch_plan(C.byref(PhgParams(20, 1, 5, 3, 0)), 481, 321, 1, None, 0) == 1
