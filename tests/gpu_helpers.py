"""Run an oracle.instances.Instance through the product path: DeviceArena
(HBM) + Runtime.launch (C ABI -> sm_100a kernel) + device_synchronize."""

from __future__ import annotations

import numpy as np

from paper_2206_07896_b200 import (ArgSlot, Average, DeviceArena, Dim3, PackedArgs, Runtime,
                                    RuntimeFault, _lib, routines)

_NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}


def registered() -> set:
    return set(_lib.kernels())


def materialize(inst, arena):
    handles = {}
    for b in inst.buffers:
        h = arena.alloc(b.scalar, b.length)
        vals = np.asarray(b.values, dtype=_NP[b.scalar]).reshape(-1)[: b.length]
        if vals.size:
            arena.upload_numpy(h, vals)
        handles[b.name] = h
    slots = [ArgSlot("handle", handles[a[1]]) if a[0] == "buf" else ArgSlot(a[0], a[1])
             for a in inst.args]
    return PackedArgs(slots), handles


def gpu_run(inst, pool_size: int = 1, policy=None, instrument: bool = False, routine=None, fetch: str = "host"):
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    if routine is None:
        routine = routines.get(inst.kernel, warp_size=inst.warp_size)
    trap = None
    with Runtime(arena, pool_size=pool_size, policy=policy or Average(), instrument=instrument,
                 fetch=fetch) as rt:
        task = rt.launch(routine, Dim3(inst.grid.x, inst.grid.y, inst.grid.z),
                         Dim3(inst.block.x, inst.block.y, inst.block.z), inst.shmem, packed)
        try:
            rt.device_synchronize()
        except RuntimeFault as e:
            trap = (e.trap.kind, e.block_id)
        counters = rt.counters
    outs = {b.name: arena.to_numpy(handles[b.name]) for b in inst.buffers}
    arena.close()  # device memory and pinned staging go now, not at interpreter exit
    return outs, trap, task, counters


def bit_equal(a: np.ndarray, b: np.ndarray) -> bool:
    return a.dtype == b.dtype and a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
