"""Host-program drivers for the graph kernel (bfs).

`bfs_levels` is Rodinia's bfs host loop (launch the level step with cur =
0, 1, ... until `changed` stays 0) fused on the device: frontier queues and
an L2-resident visited bitmap instead of a full vertex sweep per level.  It
produces exactly the levels of the per-level launches of kernels/bfs.kn
(tests/test_gpu_parity.py::test_bfs_levels_fused_vs_oracle).
"""

from __future__ import annotations

import ctypes as C
from typing import NamedTuple, Optional

from . import _lib
from ._lib import BfError


class Transposed(NamedTuple):
    """In-edge CSR of a graph (arena handles): ccol[crow[v] .. crow[v+1]) are
    the sources of the edges into v."""
    crow: int
    ccol: int


def transpose(rt, row: int, col: int, nv: int) -> Transposed:
    """Build the in-edge CSR of (row, col) on the device (bf_bfs_transpose),
    allocating its two i32 buffers in rt's arena; done once per graph."""
    arena = rt.arena
    crow = arena.alloc("i32", nv + 1)
    ccol = arena.alloc("i32", max(1, arena.length(col)))
    try:
        rc = _lib.lib().bf_bfs_transpose(rt._native, row, col, nv, crow, ccol)
        if rc != _lib.OK:
            raise BfError(rc, _lib.last_error())
    except BaseException:
        arena.free(crow)
        arena.free(ccol)
        raise
    return Transposed(crow, ccol)


def bfs_levels(rt, row: int, col: int, lvl: int, nv: int, source: int = 0,
               transposed: Optional[Transposed] = None) -> int:
    """Fill buffer `lvl` with BFS levels from `source`; returns max level + 1.
    With `transposed` (from `transpose`) the traversal is
    direction-optimizing: large frontiers are expanded bottom-up."""
    depth = C.c_int32()
    if transposed is None:
        rc = _lib.lib().bf_bfs_levels(rt._native, row, col, lvl, nv, source, C.byref(depth))
    else:
        rc = _lib.lib().bf_bfs_levels_do(rt._native, row, col, transposed.crow, transposed.ccol, lvl, nv,
                                         source, C.byref(depth))
    if rc != _lib.OK:
        raise BfError(rc, _lib.last_error())
    return depth.value


class BfsShard:
    """One rank's share of a sharded traversal (bf_bfs_shard_*): the whole
    visited bitmap and level bytes on this device, expansion of the frontier
    vertices in [vlo, vhi) only.  Driven by parallel.bfs_levels_sharded."""

    def __init__(self, rt, nv: int):
        self.rt = rt
        self.nv = nv
        self._h = C.c_void_p()
        self._call("bf_bfs_shard_create", rt._native, nv, C.byref(self._h))

    def _call(self, fn, *args):
        rc = getattr(_lib.lib(), fn)(*args)
        if rc != _lib.OK:
            raise BfError(rc, _lib.last_error())

    def bitmap(self):
        """(device pointer, uint32 word count) of the visited bitmap."""
        ptr, words = C.c_void_p(), C.c_int64()
        self._call("bf_bfs_shard_bitmap", self._h, C.byref(ptr), C.byref(words))
        return ptr.value, words.value

    def begin(self, source: int, vlo: int, vhi: int) -> None:
        self._call("bf_bfs_shard_begin", self._h, source, vlo, vhi)

    def expand(self, row: int, col: int) -> None:
        self._call("bf_bfs_shard_expand", self._h, row, col)

    def merge(self, gathered_ptr: int, world: int) -> None:
        self._call("bf_bfs_shard_merge", self._h, C.c_void_p(gathered_ptr), world)

    def bitmap_tensor(self, world: int):
        """The visited bitmap as a torch int32 device view of world x
        ceil(words / world) words (the shard pads it with 64 zero words)."""
        import torch

        from .parallel import _device_view, bitmap_slices
        if world > 64:
            raise ValueError("the bitmap padding covers at most 64 ranks")
        ptr, words = self.bitmap()
        return _device_view(ptr, world * bitmap_slices(words, world),
                            torch.device("cuda", self.rt.arena.device))

    def merge_slice(self, recv, world: int, first: int, count: int) -> None:
        """now[first + i] = OR over r of recv[r * count + i] (device tensor)."""
        self._call("bf_bfs_shard_merge_slice", self._h, C.c_void_p(recv.data_ptr()), world, first, count)

    def compact(self, lvl: int) -> int:
        fresh = C.c_int64()
        self._call("bf_bfs_shard_compact", self._h, lvl, C.byref(fresh))
        return fresh.value

    def finish(self, lvl: int) -> int:
        depth = C.c_int32()
        self._call("bf_bfs_shard_finish", self._h, lvl, C.byref(depth))
        return depth.value

    def close(self) -> None:
        if self._h:
            _lib.lib().bf_bfs_shard_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
