"""Host-program driver for the kmeans kernel (§8e kmeans
"+1 exchange/iteration").

Rodinia's kmeans_clustering loop: membership starts at -1; every pass runs
the assignment kernel (kernels/kmeans.kn: nearest centroid, plus the per
cluster feature sums and member counts), replaces each centroid that has
members by sums / counts (f32), and counts delta = points whose membership
changed; it stops when delta <= threshold or after max_iter passes
(`while (delta > threshold && loop++ < 500)`).

Across ranks (one process per GPU) each rank assigns its contiguous range of
logical blocks (parallel.rank_range), the 16 x 32 sums and 16 counts are
all-reduced (~2.1 KB per pass) before the centroid update, and delta is
all-reduced after it; every rank then holds the same centroids.

The device work is ours: the assignment kernel through Runtime.launch /
launch_range and bf_kmeans_update (centroids, clearing, delta).  The sums
are f32 sums in a different order than the reference's sequential adds
(SPEC.md:420), so centroids can differ from a sequential host loop in the
last bits and later passes may assign tied points differently; each pass's
membership is exactly the reference assignment for the centroids it used
(tests/test_gpu_parity.py::test_kmeans_iterate_*).
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Optional

from . import _lib
from ._lib import BfError


class KmeansDriver:
    """One rank's state of the host loop; `kmeans_iterate` drives it."""

    def __init__(self, rt, arena, f: int, cent: int, member: int, npts: int, nf: int, k: int,
                 world: int = 1, rank: int = 0, block: int = 256):
        from . import ArgSlot, Dim3, PackedArgs, routines
        from .parallel import rank_range
        self.rt, self.arena = rt, arena
        self.cent, self.member = cent, member
        self.npts, self.nf, self.k = npts, nf, k
        self.sums = arena.alloc("f32", k * nf)
        self.counts = arena.alloc("i32", k)
        self.prev = arena.alloc("i32", npts)
        arena.fill_value(self.prev, -1)            # Rodinia: membership[i] = -1
        self.routine = routines.get("kmeans")
        self.grid, self.block = Dim3(-(-npts // block)), Dim3(block)
        self.packed = PackedArgs([ArgSlot("handle", f), ArgSlot("handle", cent), ArgSlot("handle", member),
                                  ArgSlot("handle", self.sums), ArgSlot("handle", self.counts),
                                  ArgSlot("i32", npts), ArgSlot("i32", nf), ArgSlot("i32", k)])
        self.world, self.rank = world, rank
        self.b_lo, self.b_hi = rank_range(self.grid.x, world, rank)
        self.p_lo, self.p_hi = self.b_lo * block, min(self.b_hi * block, npts)

    def assign(self) -> None:
        if self.b_hi > self.b_lo:
            if self.world == 1:
                self.rt.launch(self.routine, self.grid, self.block, 0, self.packed)
            else:
                self.rt.launch_range(self.routine, self.grid, self.block, 0, self.packed, self.b_lo,
                                     self.b_hi - self.b_lo)
        self.rt.device_synchronize()

    def update(self) -> int:
        """Centroids from (already reduced) sums/counts; returns this rank's delta."""
        d = C.c_int64()
        rc = _lib.lib().bf_kmeans_update(self.rt._native, self.cent, self.sums, self.counts, self.nf, self.k,
                                         self.member, self.prev, self.p_lo, self.p_hi, C.byref(d))
        if rc != _lib.OK:
            raise BfError(rc, _lib.last_error())
        return d.value


def kmeans_iterate(rt, arena, f: int, cent: int, member: int, npts: int, nf: int, k: int,
                   threshold: float = 0.001, max_iter: int = 500, world: int = 1, rank: int = 0,
                   allreduce: Optional[Callable] = None) -> tuple[int, int]:
    """Run the loop; `cent` ends with the final centroids, `member` with the
    last assignment.  `allreduce(handles)` sums arena buffers over the ranks
    in place, `allreduce(int)` sums a scalar (parallel.nccl_allreduce).
    Returns (passes, last delta)."""
    drv = KmeansDriver(rt, arena, f, cent, member, npts, nf, k, world, rank)
    passes = 0
    while True:
        drv.assign()
        if world > 1:
            allreduce([drv.sums, drv.counts])
        delta = drv.update()
        if world > 1:
            delta = allreduce(delta)
        passes += 1
        if not (delta > threshold and passes < max_iter + 1):
            return passes, delta
