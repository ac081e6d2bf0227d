"""Pure-copy version of the C4 e2e pipeline (no kernels): n chunks of the
632 MB batch, H2D of chunk i+1 overlapping D2H of chunk i on separate
streams.  The ceiling the batch pipeline can reach on this host."""
import time

import torch

N = 632426496
src = torch.empty(N, dtype=torch.uint8).pin_memory()
dst = torch.empty(N, dtype=torch.uint8).pin_memory()
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
for nch in (1, 4, 8, 16, 32):
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    bounds = [N * c // nch for c in range(nch + 1)]

    def run():
        evs = []
        for c in range(nch):
            a, b = bounds[c], bounds[c + 1]
            with torch.cuda.stream(sh):
                dev[a:b].copy_(src[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(sh)
            with torch.cuda.stream(sd):
                sd.wait_event(e)
                dst[a:b].copy_(dev[a:b], non_blocking=True)
        torch.cuda.synchronize()

    run()
    t0 = time.perf_counter()
    for _ in range(5):
        run()
    ms = (time.perf_counter() - t0) / 5 * 1e3
    print(f"chunks {nch:3d}: {ms:7.2f} ms  -> {632426496 * 5 / ms / 1e3 / 1e3:8.1f} K Mpix-it/s equivalent")
