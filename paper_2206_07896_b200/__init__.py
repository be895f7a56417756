"""B200-native launch runtime and benchmark kernels for the hot path of the
reference `blockfuse` (arXiv 2206.07896, CuPBoP).

The public surface mirrors `blockfuse.runtime` / `blockfuse.arena`:

    from paper_2206_07896_b200 import DeviceArena, Runtime, Dim3, ArgSlot, PackedArgs, routines
    arena = DeviceArena()
    with Runtime(arena) as rt:
        rt.launch(routines.get("vecadd"), Dim3(4096), Dim3(256), 0, packed)
        rt.device_synchronize()

Every launch runs a hand-written sm_100a kernel from libbfgpu.so; importing
the runtime without the built library raises (no CPU fallback).
"""

from .arena import DeviceArena, Trap, wrap_int, SCALAR_SIZE
from .runtime import (
    ArgSlot,
    Average,
    AutoAggressive,
    Dim3,
    Fixed,
    KernelTask,
    PackedArgs,
    PoolShutdown,
    Runtime,
    RuntimeCounters,
    RuntimeFault,
    TaskQueue,
    delinearize,
    linearize,
    parse_policy,
    resolve_grain,
)
from . import routines
from .routines import KernelNotImplemented, Routine

__all__ = [
    "DeviceArena", "Trap", "wrap_int", "SCALAR_SIZE", "ArgSlot", "Average", "AutoAggressive",
    "Dim3", "Fixed", "KernelTask", "PackedArgs", "PoolShutdown", "Runtime", "RuntimeCounters",
    "RuntimeFault", "TaskQueue", "delinearize", "linearize", "parse_policy", "resolve_grain",
    "routines", "KernelNotImplemented", "Routine",
]
