"""Synthetic inputs for the BASELINE configs.

Generated with the reference's own generators as restated in the C++ host
library: synth_image(SmoothRandom) (image.hpp:77-103) + inject_sp_noise
(noise.hpp:62-89).  Generation is host-side and outside every timed region.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .phgrms import GrayImage, NoiseSpec, inject_sp_noise, synth_image


@dataclass(frozen=True)
class Workload:
    key: str
    width: int
    height: int
    n_images: int
    beta: int
    description: str


WORKLOADS = {
    "c1": Workload("c1", 481, 321, 1, 1, "481x321 BSDS-size, 10% s&p, beta=1, k=5"),
    "c2": Workload("c2", 3840, 2160, 1, 1, "3840x2160 (4K), 30% s&p, beta=1, k=5"),
    "c3": Workload("c3", 16384, 16384, 1, 2, "16384x16384, 50% s&p, beta=2, k=5"),
    "c4": Workload("c4", 481, 321, 4096, 1,
                   "batch of 4096 481x321 images per rank, 10-70% s&p, beta=1, k=5"),
}


def c4_density(i: int) -> float:
    """d = 0.10 + 0.60 * (i mod 61) / 60."""
    return 0.10 + 0.60 * (i % 61) / 60


def c4_image(i: int, w: int = 481, h: int = 321) -> np.ndarray:
    clean = synth_image(w, h, i)
    return inject_sp_noise(clean, NoiseSpec(c4_density(i), 0.5, i)).pixels


def make_batch(first: int, n: int, w: int = 481, h: int = 321, out: np.ndarray = None,
               threads: int = None) -> np.ndarray:
    """Images first..first+n-1 of the C4 stream, packed [n][h][w]."""
    if out is None:
        out = np.empty((n, h, w), np.uint8)
    threads = threads or min(32, os.cpu_count() or 1)

    def one(j):
        out[j] = c4_image(first + j, w, h)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, range(n)))
    return out


def single_image(key: str) -> np.ndarray:
    wl = WORKLOADS[key]
    density = {"c1": 0.10, "c2": 0.30, "c3": 0.50}[key]
    clean = synth_image(wl.width, wl.height, 1)
    return inject_sp_noise(clean, NoiseSpec(density, 0.5, 12345)).pixels


# ----------------------------------------------------------- C5 giga-pixel
C5_SIZE = 65536
C5_TILE = 4096


def c5_tile(ti: int, tj: int, tile: int = C5_TILE) -> np.ndarray:
    """Tile (ti, tj) of the C5 image.  The reference's inject_sp_noise draws
    bounded_rand(uint32(total - i)), which divides by zero at 2^32 pixels
    (SURVEY.md section 2), so the giga-pixel input is built per 4096^2 tile
    with the reference's own generators: synth_image(SmoothRandom, seed
    1 + 16*ti + tj) + inject_sp_noise(30%, salt 0.5, seed 12345 + 16*ti + tj).
    Documented as a new generator; tile seams are ordinary image
    content for the denoiser."""
    k = 16 * ti + tj
    clean = synth_image(tile, tile, 1 + k)
    return inject_sp_noise(clean, NoiseSpec(0.30, 0.5, 12345 + k)).pixels


def c5_rows(lo: int, hi: int, size: int = C5_SIZE, tile: int = C5_TILE, out: np.ndarray = None,
            threads: int = None) -> np.ndarray:
    """Global rows [lo, hi) of the C5 image (generated tile by tile)."""
    if out is None:
        out = np.empty((hi - lo, size), np.uint8)
    threads = threads or min(32, os.cpu_count() or 1)
    jobs = [(ti, tj) for ti in range(lo // tile, (hi - 1) // tile + 1) for tj in range(size // tile)]

    def one(job):
        ti, tj = job
        t = c5_tile(ti, tj, tile)
        r0, r1 = max(lo, ti * tile), min(hi, (ti + 1) * tile)
        out[r0 - lo:r1 - lo, tj * tile:(tj + 1) * tile] = t[r0 - ti * tile:r1 - ti * tile]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one, jobs))
    return out
