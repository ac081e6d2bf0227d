#!/usr/bin/env python
"""Throughput of the ops on either side of the denoise loop (SURVEY.md 8(f)
rows f1, f4), on one B200, inputs resident in HBM, CUDA-event timed on the
launching stream after warm-up; one JSON line per op.

  cardinality   phg_dev_cardinality (beta=1: fp16 two-tile sweep, int32 map)
                algorithmic bytes 1 B in + 4 B out per pixel
  residual      phg_dev_residual_count (beta=1: count C < thr, no map)
                algorithmic bytes 1 B in per pixel
  sse           phg_dev_sse (exact uint64 numerator of mse)
                algorithmic bytes 2 B in per pixel
  removal       phg_dev_removal (denoise_pass with a caller-supplied int32
                map, denoise.hpp:243-283): 1 B image + 4 B map in, 1 B out
  denoise_beta3 phg_dev_denoise, beta = 3 (7x7 windows), k = 4, on a 30%
                salt-and-pepper image (device generators): 2 B per
                pixel-iteration; the Mpixel_per_s column is pixel-iterations

Workloads: the c4 batch (4096 x 481x321 = 632 Mpx) and one 16384^2 image
(268 Mpx), both larger than L2.  Synthetic inputs (uniform random bytes):
for `removal` that is the worst case, ~2/3 of the pixels flagged by the map
(a denoise-stream map flags 10-30%).

    python bench_ops.py [--reps 20]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="", help="comma-separated op names")
    a = ap.parse_args()
    import torch

    from paper_1306_5390_b200._lib import PhgDevImage, PhgParams, check, lib

    L = lib()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"

    def dev_image(t, w, h, n):
        im = PhgDevImage()
        im.data = t.data_ptr()
        im.pitch = t.shape[-1]
        im.image_stride = t.shape[-1] * h
        im.width, im.rows, im.n_images = w, h, n
        return im

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    for wl, (n, w, h) in (("c4 batch 4096x481x321", (4096, 481, 321)), ("16384^2 image", (1, 16384, 16384))):
        pitch = (w + 15) // 16 * 16
        x = torch.randint(0, 256, (n, h, pitch), dtype=torch.uint8, device=dev)
        y = torch.randint(0, 256, (n, h, pitch), dtype=torch.uint8, device=dev)
        ix, iy = dev_image(x, w, h, n), dev_image(y, w, h, n)
        cpitch = (w + 3) // 4 * 4
        card = torch.empty((n, h, cpitch), dtype=torch.int32, device=dev)
        cnt = torch.zeros(n, dtype=torch.int64, device=dev)
        ctr = torch.zeros((n, 1, 2), dtype=torch.int64, device=dev)
        iz = dev_image(y, w, h, n)
        params = PhgParams(20, 1, 1, 3, 0)
        params2 = PhgParams(20, 2, 1, 3, 0)
        px = n * w * h
        ops = {
            "cardinality": (5.0, lambda: check(L.phg_dev_cardinality(C.byref(ix), 20, 1, C.c_void_p(card.data_ptr()),
                                                                     cpitch, sh))),
            "residual": (1.0, lambda: check(L.phg_dev_residual_count(C.byref(ix), 20, 1, 3,
                                                                     C.c_void_p(cnt.data_ptr()), sh))),
            "sse": (2.0, lambda: check(L.phg_dev_sse(C.byref(ix), C.byref(iy), C.c_void_p(cnt.data_ptr()), sh))),
            "cardinality_beta2": (5.0, lambda: check(L.phg_dev_cardinality(C.byref(ix), 20, 2,
                                                                           C.c_void_p(card.data_ptr()), cpitch, sh))),
            "removal": (6.0, lambda: check(L.phg_dev_removal(C.byref(ix), C.c_void_p(card.data_ptr()), cpitch,
                                                             C.byref(params), C.byref(iz),
                                                             C.c_void_p(ctr.data_ptr()), sh))),
            "removal_beta2": (6.0, lambda: check(L.phg_dev_removal(C.byref(ix), C.c_void_p(card.data_ptr()), cpitch,
                                                                   C.byref(params2), C.byref(iz),
                                                                   C.c_void_p(ctr.data_ptr()), sh))),
        }
        # beta = 3 denoise: clean smooth field + 30% noise (phg_dev_synth_smooth / inject)
        k3 = 4
        nz = torch.empty_like(x)
        inz = dev_image(nz, w, h, n)
        check(L.phg_dev_synth_smooth(C.byref(inz), 0, h, C.c_uint64(7), sh))
        check(L.phg_dev_inject_noise(C.byref(inz), 0, h, C.c_double(0.3), C.c_double(0.5), C.c_uint64(9), None, sh))
        ctr3 = torch.zeros((n, k3, 2), dtype=torch.int64, device=dev)
        p3 = PhgParams(20, 3, k3, 3, 0)
        ops["denoise_beta3"] = (2.0 * k3, lambda: check(L.phg_dev_denoise(C.byref(inz), C.byref(iy), C.byref(ix),
                                                                          C.byref(p3), C.c_void_p(ctr3.data_ptr()),
                                                                          sh)))
        for name, (bpp, fn) in ops.items():
            if a.only and name not in a.only.split(","):
                continue
            ms = timed(fn)
            gbs = px * bpp / (ms / 1e3) / 1e9
            units = px * (bpp / 2.0 if name.startswith("denoise") else 1.0)
            print(json.dumps({"op": name, "workload": wl, "ms": round(ms, 4), "Mpixel_per_s": round(units / ms / 1e3, 1),
                              "alg_bytes_per_px": bpp, "achieved_GBs": round(gbs, 1), "peak_GBs": peak,
                              "frac": round(gbs / peak, 4), "peak_source": peak_src,
                              "data": ("device smooth field + 30% s&p" if name.startswith("denoise")
                                       else "synthetic uniform")}))
        del x, y, card, nz


if __name__ == "__main__":
    main()
