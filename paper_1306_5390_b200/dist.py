"""Multi-GPU sharding of the denoise path (one process per GPU).

Two decompositions, both following the reference's own row_blocks formula
(lo = n*g/G, hi = n*(g+1)/G; include/phgrms/denoise.hpp:97-107):

* Batch (config C4): images are independent, so rank g takes images
  [n*g/G, n*(g+1)/G) and runs them with no data-path collective.  Per-image
  stats stay per image.

* Giga-pixel row bands (config C5): rank g owns global rows [lo, hi) of a
  single image and keeps a beta*Tmax-row halo above and below.  Every fused
  launch of T iterations (temporal blocking) is followed by one halo
  exchange: the band's first/last beta*Tmax owned rows go to the neighbours
  with torch.distributed P2P (NCCL send/recv over NVLink on the GPU path,
  gloo in the CPU tests).  Per-iteration counters are summed with ONE
  all_reduce at the end; because a zero-replacement iteration is a fixed
  point (SPEC.md "Fixed point"), running all k iterations and truncating the
  stats afterwards is bit-identical to the reference's early stop.

The band stepper is injected: on GPUs it is the C-ABI fused kernel
(``cuda_band_stepper``); the CPU tests drive the same exchange schedule with
the oracle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, List, Tuple

import torch
import torch.distributed as dist

from .phgrms import row_blocks


def shard(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[lo, hi) of rank `rank` -- the row_blocks partition (may be empty)."""
    return n * rank // world, n * (rank + 1) // world


def chunk_plan(k: int, tmax: int) -> List[int]:
    """k iterations split into ceil(k/tmax) launches, sizes as even as possible."""
    n = max(1, -(-k // max(1, tmax)))
    return [k // n + (1 if i < k % n else 0) for i in range(n)]


@dataclass
class BandPlan:
    height: int
    width: int
    world: int
    rank: int
    halo: int  # beta * Tmax rows kept on each side

    def __post_init__(self):
        blocks = row_blocks(self.height, self.world)
        if len(blocks) != self.world:
            raise ValueError("row bands: image has fewer rows than ranks")
        b = blocks[self.rank]
        self.lo, self.hi = b.begin, b.end
        if min(bb.end - bb.begin for bb in blocks) < self.halo:
            raise ValueError("row bands: every band must hold at least beta*T rows")
        self.blo = max(0, self.lo - self.halo)
        self.bhi = min(self.height, self.hi + self.halo)
        self.up = self.rank - 1 if self.rank > 0 else None
        self.down = self.rank + 1 if self.rank < self.world - 1 else None

    @property
    def rows(self) -> int:
        return self.bhi - self.blo

    def local(self, g: int) -> int:
        """buffer row of global row g"""
        return g - self.blo


def exchange_halos(buf: torch.Tensor, plan: BandPlan, group=None) -> None:
    """Refresh the halo rows of `buf` ([rows, pitch], rows = plan.rows) from
    the neighbouring bands' freshly computed owned rows.  Sends are views of
    the owned rows; receives land directly in the halo rows."""
    ops = []
    if plan.up is not None:
        h = plan.lo - plan.blo
        ops.append(dist.P2POp(dist.isend, buf[plan.local(plan.lo):plan.local(plan.lo) + h].contiguous(),
                              plan.up, group))
        ops.append(dist.P2POp(dist.irecv, _RecvSlot(buf, 0, h).tensor, plan.up, group))
    if plan.down is not None:
        h = plan.bhi - plan.hi
        ops.append(dist.P2POp(dist.isend, buf[plan.local(plan.hi) - h:plan.local(plan.hi)].contiguous(),
                              plan.down, group))
        ops.append(dist.P2POp(dist.irecv, _RecvSlot(buf, plan.local(plan.hi), h).tensor, plan.down, group))
    if not ops:
        return
    if buf.is_cuda and dist.get_backend(group) == "gloo":
        _exchange_staged(ops)  # gloo's send/recv take host tensors (CPU multi-rank tests)
        return
    for r in dist.batch_isend_irecv(ops):
        r.wait()


def _exchange_staged(ops) -> None:
    """The same P2P ops through host copies (gloo cannot send device tensors)."""
    staged = [(op, op.tensor.cpu()) for op in ops]
    reqs = [dist.P2POp(op.op, t, op.peer, op.group) for op, t in staged]
    for r in dist.batch_isend_irecv(reqs):
        r.wait()
    for op, t in staged:
        if op.op is dist.irecv:
            op.tensor.copy_(t)


class _RecvSlot:
    """Receive straight into contiguous halo rows of the band buffer."""

    def __init__(self, buf, r0, n):
        self.tensor = buf[r0:r0 + n]
        assert self.tensor.is_contiguous()


Stepper = Callable[[torch.Tensor, torch.Tensor, BandPlan, int, int], None]


def denoise_band(src: torch.Tensor, tmp_a: torch.Tensor, tmp_b: torch.Tensor, plan: BandPlan, k: int,
                 tmax: int, stepper: Stepper, group=None) -> torch.Tensor:
    """k iterations of the band pipeline.  `src` (never written) holds this
    rank's owned rows plus valid halos; the result is returned in one of
    tmp_a/tmp_b (whose halo rows are refreshed after every launch)."""
    cur, nxt = src, tmp_a
    it0 = 0
    launches = chunk_plan(k, tmax)
    for i, iters in enumerate(launches):
        stepper(cur, nxt, plan, it0, iters)
        if i + 1 < len(launches):  # the last launch's halos are never read
            exchange_halos(nxt, plan, group)
        cur = nxt
        nxt = tmp_b if nxt is tmp_a else tmp_a
        it0 += iters
    return cur


def reduce_counters(counters: torch.Tensor, group=None) -> torch.Tensor:
    """ONE all_reduce of the [k, 2] (flagged, replaced) counters."""
    dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def truncate_stats(counters) -> List[Tuple[int, int]]:
    """denoise.hpp:308 -- stop after the first zero-replacement iteration."""
    out = []
    for f, r in counters.tolist():
        out.append((int(f), int(r)))
        if r == 0:
            break
    return out


# ------------------------------------------------------------ GPU stepper
def cuda_band_stepper(params, counters: torch.Tensor, width: int, height: int, stream=None):
    """Stepper running the fused sm_100a kernel (phg_dev_fused_step) on band
    buffers that live on the current CUDA device.  counters: int64 [k, 2].
    With ``peers`` (a list of PhgHaloPeer) the launch also stores the owned
    rows that lie in the neighbours' halos into their buffers
    (phg_dev_fused_step_mirrored)."""
    from ._lib import PhgDevImage, PhgHaloPeer, check, lib

    L = lib()
    kcap = counters.shape[0]

    def step(src, dst, plan, it0, iters, peers=None):
        s = PhgDevImage(src.data_ptr(), src.stride(0), src.stride(0) * plan.rows, width, plan.rows, 1, 0)
        d = PhgDevImage(dst.data_ptr(), dst.stride(0), dst.stride(0) * plan.rows, width, plan.rows, 1, 0)
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        if peers:
            arr = (PhgHaloPeer * len(peers))(*peers)
            check(L.phg_dev_fused_step_mirrored(C.byref(s), C.byref(d), plan.blo, height, plan.lo, plan.hi,
                                                C.byref(params), it0, iters, C.c_void_p(counters.data_ptr()),
                                                kcap, arr, len(peers), C.c_void_p(st)))
        else:
            check(L.phg_dev_fused_step(C.byref(s), C.byref(d), plan.blo, height, plan.lo, plan.hi,
                                       C.byref(params), it0, iters, C.c_void_p(counters.data_ptr()), kcap,
                                       C.c_void_p(st)))

    return step


# ------------------------------------------- fused halo exchange (CUDA IPC)
def mirror_rows(plan: BandPlan, other: BandPlan) -> Tuple[int, int]:
    """Global rows of `plan`'s band that lie in the halo of the neighbouring
    band `other` ([lo, hi), possibly empty)."""
    return max(plan.lo, other.blo), min(plan.hi, other.bhi)


class IpcHaloPeers:
    """The neighbours' ping-pong band buffers mapped into this process with
    CUDA IPC (one process per GPU on an NVSwitch node), as PhgHaloPeer lists
    for the mirrored stepper: launch i of every rank writes the rows its
    neighbours need straight into their buffer i % 2 -- NVLink stores issued
    by the kernel epilogue -- so no exchange step follows the launch.

    ``bufs`` are this rank's two [rows, pitch] uint8 CUDA tensors; all ranks
    of ``group`` call the constructor (it all-gathers the handles)."""

    def __init__(self, plan: BandPlan, bufs, group=None):
        from ._lib import PhgHaloPeer, check, lib

        L = lib()
        self.L, self.plan = L, plan
        mine = []
        for b in bufs:
            h = (C.c_uint8 * 64)()
            off = C.c_uint64()
            check(L.phg_ipc_get_handle(C.c_void_p(b.data_ptr()), h, C.byref(off)))
            mine.append((bytes(h), int(off.value), int(b.stride(0))))
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, (plan.rank, plan.blo, plan.bhi, mine), group=group)
        self.opened = []
        self.peers = [[], []]  # per parity
        for nb in (plan.up, plan.down):
            if nb is None:
                continue
            rank, blo, bhi, hs = allh[nb]
            other = BandPlan(plan.height, plan.width, plan.world, rank, plan.halo)
            lo, hi = mirror_rows(plan, other)
            for parity, (hb, off, pitch) in enumerate(hs):
                if pitch != bufs[parity].stride(0):
                    raise ValueError("band buffers must share one pitch")
                ptr = C.c_void_p()
                check(L.phg_ipc_open_handle((C.c_uint8 * 64).from_buffer_copy(hb), off, C.byref(ptr)))
                self.opened.append((ptr.value, off))
                if hi > lo:
                    self.peers[parity].append(PhgHaloPeer(ptr.value, blo, lo, hi, 0))

    def for_buffer(self, parity: int):
        return self.peers[parity]

    def close(self):
        for ptr, off in self.opened:
            self.L.phg_ipc_close(C.c_void_p(ptr), off)
        self.opened = []


def denoise_band_fused(src: torch.Tensor, bufs, plan: BandPlan, k: int, tmax: int, stepper, peers: IpcHaloPeers,
                       group=None) -> torch.Tensor:
    """denoise_band with the halo exchange fused into the launches: launch i
    writes bufs[i % 2] and, through the IPC mirrors, the neighbours'
    bufs[i % 2] halo rows.  Between launches one host barrier orders launch i
    of every rank after launch i-1 of its neighbours (they read the rows the
    next launch overwrites, and write the rows it reads)."""
    cur = src
    it0 = 0
    launches = chunk_plan(k, tmax)
    for i, iters in enumerate(launches):
        if i > 0:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=group)
        last = i + 1 == len(launches)  # the last launch's halos are never read
        stepper(cur, bufs[i % 2], plan, it0, iters, None if last else peers.for_buffer(i % 2))
        cur = bufs[i % 2]
        it0 += iters
    return cur
