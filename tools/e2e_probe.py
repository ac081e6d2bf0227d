"""Where the time of one single-image host-buffer call goes (C2 shape):
pinned H2D + D2H alone, the resident kernel, and phg_denoise end to end."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1306_5390_b200 as P
from paper_1306_5390_b200._lib import PhgParams, PhgPassStats, lib

w, h = 3840, 2160
L = lib()
img = torch.randint(0, 256, (h, w), dtype=torch.uint8).pin_memory()
out = torch.empty((h, w), dtype=torch.uint8).pin_memory()
dev = torch.empty((h, w), dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def copies():
    with torch.cuda.stream(s):
        dev.copy_(img, non_blocking=True)
        out.copy_(dev, non_blocking=True)
    s.synchronize()


p = PhgParams(20, 1, 5, 3, 0)
st = (PhgPassStats * 5)()
it = C.c_int()


def den():
    L.phg_denoise(img.data_ptr(), w, h, C.byref(p), 1, out.data_ptr(), st, C.byref(it))


print("copies H2D+D2H ms", round(t(copies), 4))
print("phg_denoise ms", round(t(den), 4))
for rc in ("2", "4"):
    os.environ["PHG_ROW_CHUNKS"] = rc
print("Mpix-it/s at phg_denoise:", round(w * h * 5 / t(den) / 1e3, 1))
