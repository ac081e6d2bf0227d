#!/usr/bin/env python
"""Benchmark of the P-HGRMS denoise hot path on B200 (one process per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c2|c1|c3|c5] [--c5-size S]

Metric (BASELINE.json): Mpixel-iterations/s (and % of the HBM roofline).
A step = one full k=5 denoise of this rank's batch (default workload c4:
4096 images of 481x321 per rank, 10-70% salt & pepper, beta=1, alpha=20).

  value     whole-job Mpixel-iterations/s with inputs resident in HBM
            (phg_dev_denoise on device buffers), device-timed with CUDA
            events, max over ranks.
  e2e       the same metric through the public host-buffer C ABI
            (phg_denoise_batch from pinned host memory: H2D, kernels, D2H of
            the images and per-iteration counters inside the timed region).
  roofline  the dominant kernel (fused_h2_kernel for beta=1 / fused_h2b2_kernel for
            beta=2, T iterations per launch)
            against MEASURED_PEAKS.json hbm_gbs, algorithmic bytes = 2 B per
            pixel-iteration.
  cpu_baseline  the reference's own CPU path (oracle/_ref, compiled from the
            reference headers) on a bounded sample, rank 0, N=1 only.

--impl reference runs only the reference CPU implementation (rank 0) and
prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel-iterations/s and % of HBM roofline at 1/2/4/8 B200 vs CPU ref"
UNIT = "Mpixel-iterations/s"
ALPHA, K = 20, 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c2", "c1", "c3", "c5"])
    ap.add_argument("--c5-size", type=int, default=65536, help="c5 image side (parity runs use less)")
    ap.add_argument("--gen", default="reference", choices=["reference", "device"],
                    help="c5 input: the reference generators per 4096^2 tile on the host, or the on-device "
                         "counter-based generators (phg_dev_synth_smooth + phg_dev_inject_noise)")
    ap.add_argument("--images", type=int, default=4096, help="images per rank (c4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="images in the CPU sample (0=auto)")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------- reference arm
def cpu_reference(sample, steps, warmup, beta, threads):
    """Times the reference's own CPU path (oracle/_ref, the reference headers
    compiled in place) -- or the C oracle port when the reference could not be
    compiled -- on `sample` ([n, h, w] uint8): image-level parallelism over
    `threads` host threads for a batch, the reference's Parallel engine
    (row_blocks threads) for a single image."""
    from oracle import oracle as O

    n, h, w = sample.shape
    out = np.empty_like(sample)
    its = np.zeros(n, np.int32)
    if O.ref_available():
        kind = "reference"
        R = O.ref()
        if n > 1:
            def run():
                R.ref_denoise_batch(sample, n, w, h, ALPHA, beta, K, 3, 0, threads, out, its)
        else:
            def run():
                O.ref_denoise(sample[0], ALPHA, beta, K, 3, 0, workers=threads)
    else:
        kind = "port"
        from concurrent.futures import ThreadPoolExecutor
        ex = ThreadPoolExecutor(threads)

        def run():
            list(ex.map(lambda i: O.denoise(sample[i], ALPHA, beta), range(n)))
    for _ in range(warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = time.perf_counter() - t0
    return n * w * h * K * steps / dt / 1e6, kind, dt


def cpu_sample(a, rank=0):
    """A bounded sample of this workload for the CPU reference (~seconds)."""
    from paper_1306_5390_b200 import workloads as WL
    if a.workload == "c4":
        m = a.cpu_sample or 64
        return WL.make_batch(rank * a.images, m), f"{m} images of 481x321 (first of the rank's batch)"
    if a.workload == "c5":
        t = WL.c5_tile(0, 0, min(4096, a.c5_size))
        return t[None], f"one {t.shape[1]}x{t.shape[0]} tile of the c5 image"
    img = WL.single_image(a.workload)
    return img[None], f"the full {img.shape[1]}x{img.shape[0]} image"


def main_reference(a, rank, world):
    if rank != 0:
        return
    from paper_1306_5390_b200 import workloads as WL
    beta = 1 if a.workload in ("c4", "c5") else WL.WORKLOADS[a.workload].beta
    threads = os.cpu_count() or 1
    sample, what = cpu_sample(a)
    v, kind, dt = cpu_reference(sample, a.steps, a.warmup, beta, threads)
    desc = WL.WORKLOADS[a.workload].description if a.workload in WL.WORKLOADS else c5_desc(a)
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(dt / a.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (reference synth_image SmoothRandom + inject_sp_noise)",
            "config": {"workload": a.workload + ": " + desc, "alpha": ALPHA, "beta": beta, "k": K,
                       "parallelism": f"{threads} host threads"},
            "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": threads, "kind": kind,
                             "sample": f"{what} per step, k={K}"},
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def c5_desc(a):
    return f"{a.c5_size}x{a.c5_size} giga-pixel image, 30% s&p, beta=1, k=5, row bands over ranks"


# ------------------------------------------------------------- our arm
def dev_image(t, width, rows, n):
    from paper_1306_5390_b200._lib import PhgDevImage
    return PhgDevImage(t.data_ptr(), t.stride(-2), t.stride(0) if n > 1 else t.stride(-2) * rows, width, rows, n, 0)


class Run:
    """Common plumbing: device, distributed group, timing helpers."""

    def __init__(self, a, rank, local, world):
        import torch
        from paper_1306_5390_b200._lib import check, lib
        self.torch, self.a, self.rank, self.local, self.world = torch, a, rank, local, world
        self.L, self.check = lib(), check
        torch.cuda.set_device(local)
        check(self.L.phg_set_device(local))
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream()
        self.sh = self.stream.cuda_stream

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.world > 1:
            self.torch.distributed.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def timed(self, step, steps, warmup, flush=None):
        """Device time of `steps` calls of step(), CUDA events on the launching
        stream, max over ranks.  With `flush`, every step is timed on its own
        and L2 is flushed between steps outside the timed events."""
        torch = self.torch
        for _ in range(warmup):
            step()
        self.barrier()
        self.L.phg_reset_launch_count()
        with ClockSampler(self.local) as clk:
            if flush is None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                for _ in range(steps):
                    step()
                e1.record(self.stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
            else:
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(steps)]
                for e0, e1 in evs:
                    flush()
                    e0.record(self.stream)
                    step()
                    e1.record(self.stream)
                torch.cuda.synchronize()
                ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
        launches = int(self.L.phg_launch_count())
        ms = self.max_over_ranks(ms)
        self.barrier()
        return ms, launches, clk.summary()


def kernel_roofline(R, src, dst, counters, params, w, h, n, beta, reps, row_base=0, height=None, own=None,
                    kcap=K):
    """Average duration of the dominant kernel (one fused launch of T = k
    iterations) on the launching stream, and the roofline record."""
    torch, L = R.torch, R.L
    height = height or h
    own_lo, own_hi = own or (0, height)
    T = min(K, L.phg_max_fused_iterations(beta))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        R.check(L.phg_dev_fused_step(C.byref(src), C.byref(dst), row_base, height, own_lo, own_hi, C.byref(params),
                                     0, T, C.c_void_p(counters.data_ptr()), kcap, C.c_void_p(R.sh)))
    e0.record(R.stream)
    for _ in range(reps):
        R.check(L.phg_dev_fused_step(C.byref(src), C.byref(dst), row_base, height, own_lo, own_hi, C.byref(params),
                                     0, T, C.c_void_p(counters.data_ptr()), kcap, C.c_void_p(R.sh)))
    e1.record(R.stream)
    torch.cuda.synchronize()
    k_ms = e0.elapsed_time(e1) / reps
    alg_bytes = 2.0 * n * w * (own_hi - own_lo) * T  # 2 B per pixel-iteration
    peak, peak_src = peaks()
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(R.a.workload, {})
            if tj.get("kernel") == L.phg_fused_kernel_name(C.byref(params), T).decode():
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            pass
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
            "kernel": L.phg_fused_kernel_name(C.byref(params), T).decode(), "kernel_ms": round(k_ms, 4),
            "alg_bytes_per_launch": int(alg_bytes)}


def run_images(R, a):
    """c4 (batch, default), c1, c2, c3: whole images resident on one device."""
    torch, L = R.torch, R.L
    from paper_1306_5390_b200 import workloads as WL
    from paper_1306_5390_b200._lib import PhgParams, PhgPassStats
    wl = WL.WORKLOADS[a.workload]
    w, h, beta = wl.width, wl.height, wl.beta
    n = a.images if a.workload == "c4" else 1
    pitch = (w + 15) // 16 * 16
    params = PhgParams(ALPHA, beta, K, 3, 0)
    host_in = torch.empty((n, h, w), dtype=torch.uint8, pin_memory=True)
    hin = host_in.numpy()
    if a.workload == "c4":
        WL.make_batch(R.rank * n, n, w, h, out=hin)
    else:
        hin[0] = WL.single_image(a.workload)
    host_out = torch.empty_like(host_in).pin_memory()
    bufs = [torch.zeros((n, h, pitch), dtype=torch.uint8, device=R.dev) for _ in range(3)]
    bufs[0][:, :, :w].copy_(host_in.to(R.dev))
    src, dst, tmp = (dev_image(b, w, h, n) for b in bufs)
    counters = torch.zeros((n, K, 2), dtype=torch.int64, device=R.dev)
    resident = 3 * n * h * pitch > 126e6
    flush_buf = None if resident else torch.empty(256 << 20, dtype=torch.uint8, device=R.dev)

    def step():
        R.check(L.phg_dev_denoise(C.byref(src), C.byref(dst), C.byref(tmp), C.byref(params),
                                  C.c_void_p(counters.data_ptr()), C.c_void_p(R.sh)))

    ms, launches, clk = R.timed(step, a.steps, a.warmup, flush=(lambda: flush_buf.zero_()) if flush_buf is not None else None)
    resident_out = bufs[1][:, :, :w].cpu()  # before the roofline launches overwrite dst
    pix_it = n * w * h * K
    roof = kernel_roofline(R, src, dst, counters, params, w, h, n, beta, max(10, a.steps))

    stats = (PhgPassStats * (n * K))()
    its = (C.c_int * n)()

    def e2e_step():
        R.check(L.phg_denoise_batch(C.c_void_p(host_in.data_ptr()), n, w, h, C.byref(params),
                                    C.c_void_p(host_out.data_ptr()), stats, its))

    e2e_steps = max(3, min(a.steps, 10))
    for _ in range(2):
        e2e_step()
    R.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = R.max_over_ranks(time.perf_counter() - t0)
    same = bool(torch.equal(resident_out, host_out))
    cfg = {"workload": a.workload + ": " + wl.description, "images_per_rank": n, "width": w, "height": h,
           "alpha": ALPHA, "beta": beta, "k": K, "card_threshold": 3, "border": "Faithful",
           "global_batch": n * R.world, "parallelism": f"dp{R.world} (image shards, no collective)",
           "l2": "inputs larger than L2 (3 buffers > 126 MB)" if resident else
                 "L2 flushed between steps (256 MB write, outside the timed events)"}
    e2e = {"value": round(pix_it * R.world * e2e_steps / e2e_s / 1e6, 3), "unit": UNIT,
           "h2d_bytes_per_step": n * w * h, "d2h_bytes_per_step": n * w * h + n * K * 2 * 8,
           "path": "phg_denoise_batch (public C ABI, pinned host buffers)", "bit_identical_to_resident": same}
    return pix_it, ms, launches, clk, roof, cfg, e2e, beta


def run_bands(R, a):
    """c5: one giga-pixel image in row bands, one band per rank; a beta*T halo
    exchanged over NCCL after every fused launch (paper_1306_5390_b200/dist.py)."""
    torch, L = R.torch, R.L
    from paper_1306_5390_b200 import dist as D
    from paper_1306_5390_b200 import workloads as WL
    from paper_1306_5390_b200._lib import PhgParams
    S = a.c5_size
    beta = 1
    tmax = L.phg_max_fused_iterations(beta)
    plan = D.BandPlan(S, S, R.world, R.rank, beta * tmax)
    pitch = (S + 15) // 16 * 16
    params = PhgParams(ALPHA, beta, K, 3, 0)
    host = torch.empty((plan.rows, S), dtype=torch.uint8, pin_memory=True)
    bufs = [torch.zeros((plan.rows, pitch), dtype=torch.uint8, device=R.dev) for _ in range(3)]
    if a.gen == "device":
        gim = dev_image(bufs[0], S, plan.rows, 1)
        R.check(L.phg_dev_synth_smooth(C.byref(gim), plan.blo, S, 1, C.c_void_p(R.sh)))
        R.check(L.phg_dev_inject_noise(C.byref(gim), plan.blo, S, 0.30, 0.5, 12345, None, C.c_void_p(R.sh)))
        torch.cuda.synchronize()
        host.copy_(bufs[0][:, :S])
    else:
        WL.c5_rows(plan.blo, plan.bhi, S, min(WL.C5_TILE, S), out=host.numpy())
        bufs[0][:, :S].copy_(host.to(R.dev))
    counters = torch.zeros((K, 2), dtype=torch.int64, device=R.dev)
    stepper = D.cuda_band_stepper(params, counters, S, S, R.sh)
    group = None

    def step():
        counters.zero_()
        D.denoise_band(bufs[0], bufs[1], bufs[2], plan, K, tmax, stepper, group)

    ms, launches, clk = R.timed(step, a.steps, a.warmup)
    pix_it = (plan.hi - plan.lo) * S * K
    src = dev_image(bufs[0], S, plan.rows, 1)
    dst = dev_image(bufs[1], S, plan.rows, 1)
    roof = kernel_roofline(R, src, dst, counters, params, S, plan.rows, 1, beta, max(5, min(a.steps, 10)),
                           row_base=plan.blo, height=S, own=(plan.lo, plan.hi))
    # e2e: pinned host band -> device -> k iterations with halo exchange -> owned rows + stats back
    host_out = torch.empty((plan.hi - plan.lo, S), dtype=torch.uint8, pin_memory=True)

    if R.world == 1:
        # one rank holds the whole image: the public host-buffer C ABI call
        # (phg_denoise; row-pipelined copies for images >= 32 MB)
        from paper_1306_5390_b200._lib import PhgPassStats
        e2e_stats, e2e_its = (PhgPassStats * K)(), C.c_int()
        host_c = host.contiguous()

        def e2e_step():
            R.check(L.phg_denoise(C.c_void_p(host_c.data_ptr()), S, S, C.byref(params), 1,
                                  C.c_void_p(host_out.data_ptr()), e2e_stats, C.byref(e2e_its)))
        e2e_path = "phg_denoise (public C ABI, pinned host buffers, row-pipelined copies)"
    else:
        def e2e_step():
            bufs[0][:, :S].copy_(host, non_blocking=True)
            counters.zero_()
            out = D.denoise_band(bufs[0], bufs[1], bufs[2], plan, K, tmax, stepper, group)
            host_out.copy_(out[plan.local(plan.lo):plan.local(plan.hi), :S], non_blocking=True)
            D.reduce_counters(counters)
            counters.cpu()
            torch.cuda.synchronize()
        e2e_path = "dist.denoise_band with the C-ABI stepper, pinned host band"

    e2e_steps = max(2, min(a.steps, 5))
    e2e_step()
    R.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_s = R.max_over_ranks(time.perf_counter() - t0)
    cfg = {"workload": "c5: " + c5_desc(a), "width": S, "height": S, "alpha": ALPHA, "beta": beta, "k": K,
           "card_threshold": 3, "border": "Faithful", "band_rows_per_rank": plan.hi - plan.lo,
           "halo_rows": beta * tmax, "parallelism": f"row bands x{R.world}, NCCL halo send/recv per launch",
           "l2": "inputs larger than L2",
           "generator": ("on-device counter-based generators (kernel_gen.cuh, DESIGN.md)" if a.gen == "device"
                         else "per-4096^2-tile reference generators (DESIGN.md)")}
    e2e = {"value": round(pix_it * R.world * e2e_steps / e2e_s / 1e6, 3), "unit": UNIT,
           "h2d_bytes_per_step": plan.rows * S, "d2h_bytes_per_step": (plan.hi - plan.lo) * S + K * 2 * 8,
           "path": e2e_path}
    return pix_it, ms, launches, clk, roof, cfg, e2e, beta


def main_ours(a, rank, local, world):
    R = Run(a, rank, local, world)
    if a.workload == "c5":
        pix_it, ms, launches, clk, roof, cfg, e2e, beta = run_bands(R, a)
    else:
        pix_it, ms, launches, clk, roof, cfg, e2e, beta = run_images(R, a)
    value = pix_it * world * a.steps / (ms / 1e3) / 1e6
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        sample, what = cpu_sample(a)
        threads = os.cpu_count() or 1
        v, kind, _ = cpu_reference(sample, 2, 1, beta, threads)
        cpu = {"value": round(v, 3), "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{what} x 2 reps, k={K}, {threads} host threads"}
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": round(ms / a.steps, 4), "higher_is_better": True,
                "scaling": "strong" if a.workload == "c5" else "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (reference synth_image SmoothRandom + inject_sp_noise, per-rank seeds)",
                "config": cfg, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk,
                "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    if world > 1:
        R.torch.distributed.barrier()
        R.torch.distributed.destroy_process_group()


def main():
    a = parse()
    rank, local, world = dist_env()
    if a.impl == "reference":
        main_reference(a, rank, world)
    else:
        main_ours(a, rank, local, world)


if __name__ == "__main__":
    main()
