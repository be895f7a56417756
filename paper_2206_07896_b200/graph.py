"""Host-program drivers for the graph kernel (bfs).

`bfs_levels` is Rodinia's bfs host loop (launch the level step with cur =
0, 1, ... until `changed` stays 0) fused on the device: frontier queues and
an L2-resident visited bitmap instead of a full vertex sweep per level.  It
produces exactly the levels of the per-level launches of kernels/bfs.kn
(tests/test_gpu_parity.py::test_bfs_levels_fused_vs_oracle).
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import BfError


def bfs_levels(rt, row: int, col: int, lvl: int, nv: int, source: int = 0) -> int:
    """Fill buffer `lvl` with BFS levels from `source`; returns max level + 1."""
    depth = C.c_int32()
    rc = _lib.lib().bf_bfs_levels(rt._native, row, col, lvl, nv, source, C.byref(depth))
    if rc != _lib.OK:
        raise BfError(rc, _lib.last_error())
    return depth.value
