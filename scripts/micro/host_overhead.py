"""Host-side cost of the per-level pieces of a Rodinia-style host loop
(fill the changed flag, launch, device_synchronize, read the flag), on a
tiny graph so the kernels take ~nothing."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines

arena = DeviceArena()
nv = 1024
row = arena.alloc("i32", nv + 1); col = arena.alloc("i32", nv * 2); lvl = arena.alloc("i32", nv); chg = arena.alloc("i32", 1)
arena.upload_numpy(row, (np.arange(nv + 1) * 2).astype(np.int32))
arena.upload_numpy(col, np.random.default_rng(0).integers(0, nv, nv * 2).astype(np.int32))
lv = np.full(nv, -1, np.int32); lv[0] = 0
arena.upload_numpy(lvl, lv)
routine = routines.get("bfs")
out = np.zeros(1, np.int32)
N = 2000

def t(name, fn):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N): fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    print(f"{name:40s} {dt:8.2f} us")

with Runtime(arena) as rt:
    pk = PackedArgs([ArgSlot("handle", row), ArgSlot("handle", col), ArgSlot("handle", lvl),
                     ArgSlot("handle", chg), ArgSlot("i32", nv), ArgSlot("i32", 5)])
    t("fill_value", lambda: arena.fill_value(chg, 0))
    t("PackedArgs build", lambda: PackedArgs([ArgSlot("handle", row), ArgSlot("handle", col), ArgSlot("handle", lvl),
                     ArgSlot("handle", chg), ArgSlot("i32", nv), ArgSlot("i32", 5)]))
    t("launch (no sync)", lambda: rt.launch(routine, Dim3(nv // 256), Dim3(256), 0, pk))
    rt.device_synchronize()
    t("device_synchronize (idle)", rt.device_synchronize)
    t("launch + sync", lambda: (rt.launch(routine, Dim3(nv // 256), Dim3(256), 0, pk), rt.device_synchronize()))
    t("download 1 elem", lambda: arena.download_into(chg, out))
    t("to_numpy 1 elem", lambda: arena.to_numpy(chg))
    def level():
        arena.fill_value(chg, 0)
        rt.launch(routine, Dim3(nv // 256), Dim3(256), 0, pk)
        rt.device_synchronize()
        return int(arena.to_numpy(chg)[0])
    t("full level (fill, launch, sync, read)", level)

# vecadd PR1 launch costs: through Runtime.launch, and the bare C ABI call
import ctypes as C
from paper_2206_07896_b200 import _lib
from paper_2206_07896_b200.runtime import pack_slots
n = 1 << 20
h = [arena.alloc("f32", n) for _ in range(3)]
pk = PackedArgs([ArgSlot("handle", h[0]), ArgSlot("handle", h[1]), ArgSlot("handle", h[2]), ArgSlot("i32", n)])
va = routines.get("vecadd")
with Runtime(arena) as rt:
    t("vecadd launch (Runtime.launch, no sync)", lambda: rt.launch(va, Dim3(4096), Dim3(256), 0, pk))
    rt.device_synchronize()
    slots, ns = pack_slots(pk)
    g = (C.c_int32 * 3)(4096, 1, 1); b = (C.c_int32 * 3)(256, 1, 1); tid = C.c_uint64()
    L = _lib.lib()
    t("vecadd launch (bf_launch via ctypes)", lambda: L.bf_launch(rt._native, b"vecadd", g, b, 0, slots, ns, 32, 4096, C.byref(tid)))
    rt.device_synchronize()
    t("vecadd launch + sync", lambda: (rt.launch(va, Dim3(4096), Dim3(256), 0, pk), rt.device_synchronize()))
    torch.cuda.synchronize()
    s = torch.cuda.ExternalStream(rt.worker_stream(0))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for rep in range(3):
        ev[0].record(s)
        for _ in range(200): rt.launch(va, Dim3(4096), Dim3(256), 0, pk)
        ev[1].record(s); rt.device_synchronize(); ev[1].synchronize()
        print("200 back-to-back vecadd PR1 launches: device us per launch", ev[0].elapsed_time(ev[1]) * 1e3 / 200)
