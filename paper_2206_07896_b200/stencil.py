"""Host-program driver for the stencil kernel (hotspot).

`hotspot_run` is Rodinia's hotspot host loop — `iterations` ping-pong
launches of kernels/hotspot.kn — fused on the device with temporal blocking
(several iterations per pass through HBM, each intermediate rounded to f32
exactly like the per-launch store).  Bit-identical to the launch loop
(tests/test_gpu_parity.py::test_hotspot_run_fused_vs_oracle).
"""

from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import BfError


def hotspot_run(rt, src: int, power: int, dst: int, rows: int, cols: int, params: dict,
                iterations: int, tsteps: int = 0) -> int:
    """Run `iterations` steps; returns the handle holding the result (src for
    an even count, dst for an odd one — as the launch loop)."""
    kc = (C.c_double * 5)(params["sdc"], params["rx1"], params["ry1"], params["rz1"], params["amb"])
    rc = _lib.lib().bf_hotspot_run(rt._native, src, power, dst, rows, cols, kc, iterations, tsteps)
    if rc != _lib.OK:
        raise BfError(rc, _lib.last_error())
    return src if iterations % 2 == 0 else dst
