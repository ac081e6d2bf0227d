#!/usr/bin/env python
"""Device time of phg_dev_denoise (k=5, beta=1, 30% s&p) for square images of
several sides: run once with the default launch plan and once with PHG_TMAX=1
(the T=1 launches then take the single-buffer DIRECT form on wide regions).
    python tools/tmax_probe.py SIDE [SIDE ...]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1306_5390_b200._lib import PhgDevImage, PhgParams, check, lib  # noqa: E402


def main():
    L = lib()
    st = torch.cuda.current_stream().cuda_stream
    for side in (int(s) for s in sys.argv[1:]):
        w = h = side
        pitch = (w + 15) // 16 * 16
        bufs = [torch.zeros((h, pitch), dtype=torch.uint8, device="cuda") for _ in range(3)]
        g = torch.Generator(device="cuda").manual_seed(side)
        base = torch.randint(90, 110, (h, pitch), dtype=torch.uint8, device="cuda", generator=g)
        noise = torch.rand((h, pitch), device="cuda", generator=g)
        base[noise < 0.15] = 0
        base[(noise >= 0.15) & (noise < 0.3)] = 255
        bufs[0].copy_(base)
        im = [PhgDevImage(b.data_ptr(), pitch, pitch * h, w, h, 1, 0) for b in bufs]
        ctr = torch.zeros(10, dtype=torch.int64, device="cuda")
        p = PhgParams(20, 1, 5, 3, 0)

        def run():
            check(L.phg_dev_denoise(C.byref(im[0]), C.byref(im[1]), C.byref(im[2]), C.byref(p),
                                    C.c_void_p(ctr.data_ptr()), C.c_void_p(st)))
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, int(2e9 / (w * h)))
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"TMAX={os.environ.get('PHG_TMAX', '-')} side={side} ms={ms:.4f} "
              f"Mpix-it/s={w * h * 5 / ms / 1e3:.0f}", flush=True)


if __name__ == "__main__":
    main()
