"""Python mirror of the reference's C++ API (namespace ``phgrms``), backed by
the sm_100a kernels through the C ABI.  Names, argument meaning, defaults and
error behaviour follow /root/reference/proj/include/phgrms/denoise.hpp and
image.hpp, so parity tests read like the reference's own Catch2 tests.

Every compute call runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, List, Sequence, Tuple

import numpy as np

from ._lib import InvalidArgument, PhgParams, PhgPassStats, check, lib


# ------------------------------------------------------------ value types
class BorderMode(enum.IntEnum):
    """denoise.hpp:27-30"""
    Faithful = 0
    InBounds = 1


class EngineMode(enum.IntEnum):
    """denoise.hpp:32.  On this framework both modes run on the GPU:
    Serial = one whole-image fused pipeline; Parallel(W) = W row bands
    (row_blocks partition) with halo exchange between them, the single
    device stand-in for the multi-GPU band sharding."""
    Serial = 0
    Parallel = 1


@dataclass
class DenoiseParams:
    """denoise.hpp:34-52"""
    alpha: int = 20
    beta: int = 1
    max_iterations: int = 5
    card_threshold: int = 3
    border: BorderMode = BorderMode.Faithful

    def validate(self) -> None:
        check(lib().phg_validate_params(C.byref(self._c())))

    def window_cells(self) -> int:
        return (2 * self.beta + 1) * (2 * self.beta + 1)

    def _c(self) -> PhgParams:
        return PhgParams(int(self.alpha), int(self.beta), int(self.max_iterations),
                         int(self.card_threshold), int(self.border))


@dataclass
class EngineSpec:
    """denoise.hpp:54-69"""
    mode: EngineMode = EngineMode.Serial
    workers: int = 0

    @staticmethod
    def serial() -> "EngineSpec":
        return EngineSpec(EngineMode.Serial, 1)

    @staticmethod
    def parallel(workers: int = 0) -> "EngineSpec":
        return EngineSpec(EngineMode.Parallel, workers)

    def resolved_workers(self) -> int:
        if self.mode == EngineMode.Serial:
            return 1
        if self.workers >= 1:
            return self.workers
        return max(1, os.cpu_count() or 1)


@dataclass
class PassStats:
    """denoise.hpp:71-76"""
    iteration: int = 0
    flagged: int = 0
    replaced: int = 0
    elapsed_ms: float = 0.0


class GrayImage:
    """image.hpp:16-51 -- uint8 row-major raster, index r*width+c."""

    def __init__(self, width: int, height: int, fill=0):
        if width < 1 or height < 1:
            raise InvalidArgument("image dimensions must be >= 1")
        self.width, self.height = int(width), int(height)
        if isinstance(fill, (np.ndarray, list, tuple, bytes)):
            px = np.asarray(fill, dtype=np.uint8).reshape(-1)
            if px.size != self.width * self.height:
                raise InvalidArgument("pixel count does not match dimensions")
            self.pixels = np.ascontiguousarray(px.reshape(self.height, self.width))
        else:
            self.pixels = np.full((self.height, self.width), int(fill), np.uint8)

    @staticmethod
    def from_array(a) -> "GrayImage":
        a = np.asarray(a, np.uint8)
        return GrayImage(a.shape[1], a.shape[0], a)

    def size(self) -> int:
        return self.width * self.height

    def index(self, r: int, c: int) -> int:
        return r * self.width + c

    def at(self, r: int, c: int) -> int:
        return int(self.pixels[r, c])

    def set(self, r: int, c: int, v: int) -> None:
        self.pixels[r, c] = v

    def same_shape(self, o: "GrayImage") -> bool:
        return self.width == o.width and self.height == o.height

    def copy(self) -> "GrayImage":
        return GrayImage(self.width, self.height, self.pixels.copy())

    def __eq__(self, o) -> bool:
        return isinstance(o, GrayImage) and self.same_shape(o) and bool(np.array_equal(self.pixels, o.pixels))

    def __repr__(self) -> str:
        return f"GrayImage({self.width}x{self.height})"


@dataclass
class CardinalityMap:
    """denoise.hpp:78-86"""
    width: int = 0
    height: int = 0
    counts: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def at(self, r: int, c: int) -> int:
        return int(self.counts[r * self.width + c])


@dataclass
class DenoiseResult:
    """denoise.hpp:285-288"""
    image: GrayImage
    stats: List[PassStats]


@dataclass
class RowBlock:
    begin: int = 0
    end: int = 0


class SynthKind(enum.IntEnum):
    Gradient = 0
    Checker = 1
    SmoothRandom = 2


# ------------------------------------------------- host-side helpers
def similar(a: int, b: int, alpha: int) -> bool:
    """denoise.hpp:88 -- |a-b| < alpha."""
    return abs(int(a) - int(b)) < alpha


def rms_replacement(sum_sq: int, flag: int) -> int:
    """denoise.hpp:163-169 -- llround(sqrt(sum/flag)) clamped to [0,255],
    evaluated with the exact integer rule the kernels use: the largest u with
    (2u-1)^2 * flag <= 4 * sum (or 0)."""
    import math
    u = math.isqrt(4 * sum_sq // flag) // 2 + 2  # >= the answer; walk down
    while u >= 1 and (2 * u - 1) ** 2 * flag > 4 * sum_sq:
        u -= 1
    return min(max(u, 0), 255)


def row_blocks(height: int, workers: int) -> List[RowBlock]:
    """denoise.hpp:97-107 -- contiguous non-empty blocks covering [0,height)."""
    if height < 0 or workers < 1:
        raise InvalidArgument("row_blocks: bad height or worker count")
    out = []
    for w in range(workers):
        lo, hi = height * w // workers, height * (w + 1) // workers
        if hi > lo:
            out.append(RowBlock(lo, hi))
    return out


def parallel_for_rows(height: int, workers: int, fn: Callable[[int, int], None]) -> None:
    """denoise.hpp:113-135 -- one host thread per block; join; rethrow."""
    blocks = row_blocks(height, workers)
    if len(blocks) <= 1:
        for b in blocks:
            fn(b.begin, b.end)
        return
    errors: List[BaseException] = [None] * len(blocks)

    def run(i, b):
        try:
            fn(b.begin, b.end)
        except BaseException as e:  # noqa: BLE001 - rethrown below
            errors[i] = e

    ts = [threading.Thread(target=run, args=(i, b)) for i, b in enumerate(blocks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errors:
        if e is not None:
            raise e


def synth_image(width: int, height: int, seed: int, kind: SynthKind = SynthKind.SmoothRandom) -> GrayImage:
    """image.hpp:53-106 (restated in the C++ host library)."""
    out = np.empty((height, width), np.uint8) if width >= 1 and height >= 1 else np.empty(0, np.uint8)
    check(lib().phg_synth_image(width, height, seed & 0xFFFFFFFF, int(kind), out))
    return GrayImage(width, height, out)


@dataclass
class NoiseSpec:
    density: float = 0.0
    salt_ratio: float = 0.5
    seed: int = 0


def inject_sp_noise(img: GrayImage, spec: NoiseSpec, with_mask: bool = False):
    """noise.hpp:62-89 (restated in the C++ host library)."""
    out = np.empty_like(img.pixels)
    mask = np.empty_like(img.pixels) if with_mask else None
    rc = lib().phg_inject_sp_noise(img.pixels, img.width, img.height, spec.density, spec.salt_ratio,
                                   spec.seed & 0xFFFFFFFF, out, mask.ctypes.data if with_mask else None)
    if rc < 0:
        check(int(rc))
    noisy = GrayImage(img.width, img.height, out)
    return (noisy, mask) if with_mask else noisy


# ----------------------------------------------------------- the hot path
def compute_cardinality(img: GrayImage, alpha: int, beta: int,
                        engine: EngineSpec = None) -> CardinalityMap:
    """denoise.hpp:227-241 (engine accepted for signature parity; the count is
    partition-invariant and always computed on the GPU)."""
    counts = np.empty(img.size(), np.int32)
    check(lib().phg_cardinality(img.pixels, img.width, img.height, int(alpha), int(beta), counts))
    return CardinalityMap(img.width, img.height, counts)


def denoise_pass(img: GrayImage, card: CardinalityMap, params: DenoiseParams,
                 engine: EngineSpec = None) -> Tuple[GrayImage, PassStats]:
    """denoise.hpp:243-283 -- removal with the caller-supplied map."""
    counts = np.ascontiguousarray(np.asarray(card.counts, np.int32).reshape(-1))
    if counts.size != card.width * card.height:
        raise InvalidArgument("cardinality map does not match image")
    out = np.empty_like(img.pixels)
    st = PhgPassStats()
    p = params._c()
    check(lib().phg_denoise_pass(img.pixels, img.width, img.height, counts, card.width, card.height,
                                 C.byref(p), out, C.byref(st)))
    return GrayImage(img.width, img.height, out), PassStats(1, st.flagged, st.replaced, st.elapsed_ms)


def denoise(img: GrayImage, params: DenoiseParams, engine: EngineSpec = None) -> DenoiseResult:
    """denoise.hpp:292-311.  EngineSpec.parallel(W) runs W row bands."""
    engine = engine or EngineSpec.serial()
    params.validate()
    k = params.max_iterations
    out = np.empty_like(img.pixels)
    stats = (PhgPassStats * k)()
    it = C.c_int()
    p = params._c()
    bands = engine.resolved_workers()
    check(lib().phg_denoise(img.pixels.ctypes.data, img.width, img.height, C.byref(p), bands,
                            out.ctypes.data, stats, C.byref(it)))
    return DenoiseResult(GrayImage(img.width, img.height, out),
                         [PassStats(s.iteration, s.flagged, s.replaced, s.elapsed_ms) for s in stats[: it.value]])


def denoise_batch(imgs: np.ndarray, params: DenoiseParams):
    """Batch extension: ``imgs`` is uint8 [n, h, w]; returns (images [n,h,w],
    list of per-image PassStats lists).  Bit-identical to calling denoise()
    on every image."""
    params.validate()
    imgs = np.ascontiguousarray(imgs, np.uint8)
    n, h, w = imgs.shape
    k = params.max_iterations
    out = np.empty_like(imgs)
    stats = (PhgPassStats * (n * k))()
    its = (C.c_int * n)()
    p = params._c()
    check(lib().phg_denoise_batch(imgs.ctypes.data, n, w, h, C.byref(p), out.ctypes.data, stats, its))
    per = [[PassStats(s.iteration, s.flagged, s.replaced, s.elapsed_ms) for s in stats[i * k: i * k + its[i]]]
           for i in range(n)]
    return out, per


def denoise_sharded(imgs: np.ndarray, params: DenoiseParams, devices):
    """The Parallel engine with GPUs as workers, from one process
    (phg_denoise_sharded; denoise.hpp:97-135): ``imgs`` is uint8 [h, w] (one
    image, row bands over ``devices`` with halo exchange) or [n, h, w] (image
    shards).  Returns (images, per-image PassStats lists) like denoise_batch;
    bit-identical to denoise() for every device list."""
    params.validate()
    imgs = np.ascontiguousarray(imgs, np.uint8)
    single = imgs.ndim == 2
    batch = imgs[None] if single else imgs
    n, h, w = batch.shape
    k = params.max_iterations
    out = np.empty_like(batch)
    stats = (PhgPassStats * (n * k))()
    its = (C.c_int * n)()
    devs = (C.c_int * max(1, len(devices)))(*[int(d) for d in devices])
    p = params._c()
    check(lib().phg_denoise_sharded(batch.ctypes.data, n, w, h, C.byref(p), devs, len(devices),
                                    out.ctypes.data, stats, its))
    per = [[PassStats(s.iteration, s.flagged, s.replaced, s.elapsed_ms) for s in stats[i * k: i * k + its[i]]]
           for i in range(n)]
    return (out[0], per[0]) if single else (out, per)


def residual_noise_count(img: GrayImage, alpha: int, beta: int, card_threshold: int) -> int:
    """metrics.hpp:52-59 -- pixels whose cardinality is below the threshold
    (beta = 1: counted by the fp16 two-tile sweep, no map is written)."""
    n = C.c_uint64(0)
    a = np.ascontiguousarray(img.pixels, dtype=np.uint8)
    check(lib().phg_residual_noise_count(a.ctypes.data, img.width, img.height, int(alpha), int(beta),
                                         int(card_threshold), C.byref(n)))
    return int(n.value)


@dataclass
class PsnrValue:
    """metrics.hpp:18-22 -- +inf when the images are identical."""
    decibels: float = 0.0

    def infinite(self) -> bool:
        return math.isinf(self.decibels)


def mse(a: GrayImage, b: GrayImage) -> float:
    """metrics.hpp:25-35 -- exact uint64 sum of squared differences on the
    device (sse_kernel), one final double division."""
    if not a.same_shape(b):
        raise InvalidArgument("mse: image dimensions differ")
    s = C.c_uint64(0)
    pa = np.ascontiguousarray(a.pixels, dtype=np.uint8)
    pb = np.ascontiguousarray(b.pixels, dtype=np.uint8)
    check(lib().phg_sse(pa.ctypes.data, pb.ctypes.data, a.width, a.height, C.byref(s)))
    return float(s.value) / float(a.size())


def psnr(a: GrayImage, b: GrayImage) -> PsnrValue:
    """metrics.hpp:37-42"""
    m = mse(a, b)
    if m == 0.0:
        return PsnrValue(math.inf)
    return PsnrValue(10.0 * math.log10(255.0 * 255.0 / m))


def format_db(v: PsnrValue) -> str:
    """metrics.hpp:44-50 -- 3 decimals, "inf" for identical images."""
    return "inf" if v.infinite() else "%.3f" % v.decibels


def write_p2(width: int, height: int, values, maxval: int) -> str:
    """pgm.hpp:123-136 -- the cardinality-map P2 writer of `phgrms cardmap`
    (tools/phgrms_main.cpp:151-168)."""
    v = np.asarray(values, dtype=np.int64).reshape(height, width)
    rows = [" ".join(map(str, r)) for r in v.tolist()]
    return "P2\n%d %d\n%d\n" % (width, height, maxval) + "".join(r + "\n" for r in rows)


def cardmap(img: GrayImage, alpha: int = 20, beta: int = 1) -> str:
    """`phgrms cardmap` (tools/phgrms_main.cpp:151-168): the P2 dump of
    compute_cardinality with maxval = (2 beta + 1)^2."""
    card = compute_cardinality(img, alpha, beta)
    return write_p2(card.width, card.height, card.counts, (2 * beta + 1) * (2 * beta + 1))


def denoise_pgm_file(in_path: str, out_path: str, params: DenoiseParams = None) -> List[PassStats]:
    """Denoise a binary PGM file into a P5 file with the file reads and writes
    overlapped with the host<->device copies (phg_denoise_pgm_file, SURVEY.md
    8(f) f4); the written file is the reference's write_pgm of the result
    (pgm.hpp:142-150).  Returns the per-iteration stats."""
    params = params or DenoiseParams()
    params.validate()
    k = params.max_iterations
    stats = (PhgPassStats * k)()
    it = C.c_int()
    p = params._c()
    check(lib().phg_denoise_pgm_file(os.fsencode(in_path), os.fsencode(out_path), C.byref(p), stats,
                                     C.byref(it)))
    return [PassStats(s.iteration, s.flagged, s.replaced, s.elapsed_ms) for s in stats[: it.value]]


def kernel_name(params: DenoiseParams, iters: int) -> str:
    """Which sm_100a kernel a fused launch of `iters` iterations runs for
    these parameters (phg_fused_kernel_name)."""
    return lib().phg_fused_kernel_name(C.byref(params._c()), int(iters)).decode()
