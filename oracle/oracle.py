"""ctypes wrapper of the CPU oracle (oracle.c).  TEST INFRASTRUCTURE ONLY.

`run(instance)` executes one launch of an `instances.Instance` with the
reference's lockstep semantics and returns `(outputs, trap)`: outputs maps
every buffer name to its final numpy array; trap is None or (kind, block).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}
TRAP_NAMES = {1: "OutOfBounds", 2: "DivByZero", 3: "TypeFault", 4: "NonUniformTrip"}


class Geom(C.Structure):
    _fields_ = [("gx", C.c_int), ("gy", C.c_int), ("gz", C.c_int),
                ("bx", C.c_int), ("by", C.c_int), ("bz", C.c_int)]


class OTrap(C.Structure):
    _fields_ = [("kind", C.c_int), ("pad", C.c_int), ("block", C.c_longlong)]


def build() -> Path:
    """Compile liboracle.so (make; gcc with -ffp-contract=off)."""
    src = HERE / "oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
    return _lib


def _arr(b) -> np.ndarray:
    a = np.array(b.values, dtype=_NP[b.scalar]).reshape(-1)
    if a.size < b.length:  # fill semantics: unspecified tail stays zero
        a = np.concatenate([a, np.zeros(b.length - a.size, a.dtype)])
    return np.ascontiguousarray(a[: b.length])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def run(inst, nthreads: int = 1, block_range=None):
    """block_range=(first, count): run only those logical blocks."""
    L = lib()
    if block_range is None:
        L.or_set_range(C.c_longlong(0), C.c_longlong(-1))
    else:
        L.or_set_range(C.c_longlong(block_range[0]), C.c_longlong(block_range[1]))
    bufs = {b.name: _arr(b) for b in inst.buffers}
    g = Geom(inst.grid.x, inst.grid.y, inst.grid.z, inst.block.x, inst.block.y, inst.block.z)
    t = OTrap()
    # positional values: buffers -> (ptr, len); scalars -> python values
    argv = []
    for a in inst.args:
        if a[0] == "buf":
            arr = bufs[a[1]]
            argv.append(_ptr(arr))
            argv.append(C.c_longlong(arr.size))
        elif a[0] in ("i32",):
            argv.append(C.c_int(int(a[1])))
        elif a[0] == "i64":
            argv.append(C.c_longlong(int(a[1])))
        else:
            argv.append(C.c_double(float(a[1])))
    k = inst.kernel
    fn = getattr(L, "or_" + k)
    extra = []
    if k == "kmeans" and nthreads > 1:  # membership/counts exact, sums within rounding
        fn = L.or_kmeans_mt
        extra = [C.c_int(nthreads)]
    if k == "reverse":
        extra = [C.c_longlong(inst.shmem)]
    elif k == "wreduce":
        extra = [C.c_int(inst.warp_size)]
    elif k in ("hotspot", "nn"):
        extra = [C.c_int(nthreads)]
    fn(g, *argv, *extra, C.byref(t))
    trap = None if t.kind == 0 else (TRAP_NAMES.get(t.kind, "?"), t.block)
    return bufs, trap


# buffers that several blocks accumulate into (atomic adds / flag stores):
# each host thread of run_par gets a private zeroed copy, summed afterwards
ACCUMULATE = {"hist": ("counts",), "wreduce": ("out",), "kmeans": ("sums", "counts"), "bfs": ("changed",)}


def run_par(inst, nthreads: int):
    """The launch split into `nthreads` contiguous logical-block ranges run
    concurrently on host threads (the reference's own worker-pool execution,
    runtime.py:305-350, with the average grain): ctypes releases the GIL, the
    block range is thread-local in oracle.c.  Disjoint outputs are shared;
    accumulated buffers (ACCUMULATE) are private per thread and added in
    thread order (integers: exact; kmeans f32 sums: within rounding); the
    bfs `changed` flag is OR-ed.  Returns (outputs, trap) like run()."""
    import concurrent.futures as cf
    G = inst.grid.x * inst.grid.y * inst.grid.z
    nthreads = max(1, min(nthreads, G))
    if nthreads == 1:
        return run(inst)
    L = lib()
    bufs = {b.name: _arr(b) for b in inst.buffers}
    acc = ACCUMULATE.get(inst.kernel, ())
    g = Geom(inst.grid.x, inst.grid.y, inst.grid.z, inst.block.x, inst.block.y, inst.block.z)
    fn = getattr(L, "or_" + inst.kernel)
    extra = []
    if inst.kernel == "reverse":
        extra = [C.c_longlong(inst.shmem)]
    elif inst.kernel == "wreduce":
        extra = [C.c_int(inst.warp_size)]
    elif inst.kernel in ("hotspot", "nn"):
        extra = [C.c_int(1)]
    cuts = [G * i // nthreads for i in range(nthreads + 1)]
    priv = [{name: np.zeros_like(bufs[name]) for name in acc} for _ in range(nthreads)]

    def work(i):
        L.or_set_range(C.c_longlong(cuts[i]), C.c_longlong(cuts[i + 1] - cuts[i]))
        argv = []
        for a in inst.args:
            if a[0] == "buf":
                arr = priv[i][a[1]] if a[1] in acc else bufs[a[1]]
                argv += [_ptr(arr), C.c_longlong(arr.size)]
            elif a[0] == "i32":
                argv.append(C.c_int(int(a[1])))
            elif a[0] == "i64":
                argv.append(C.c_longlong(int(a[1])))
            else:
                argv.append(C.c_double(float(a[1])))
        t = OTrap()
        fn(g, *argv, *extra, C.byref(t))
        L.or_set_range(C.c_longlong(0), C.c_longlong(-1))
        return None if t.kind == 0 else (TRAP_NAMES.get(t.kind, "?"), t.block)

    with cf.ThreadPoolExecutor(nthreads) as ex:
        traps = list(ex.map(work, range(nthreads)))
    for name in acc:
        base = bufs[name]
        if inst.kernel == "bfs":
            base |= np.bitwise_or.reduce([p[name] for p in priv])
        elif base.dtype == np.float32:
            for p in priv:
                base[:] = (base.astype(np.float64) + p[name]).astype(np.float32)
        else:
            tot = base.astype(np.int64) + sum(p[name].astype(np.int64) for p in priv)
            base[:] = ((tot + 2**31) % 2**32 - 2**31).astype(base.dtype)
    hit = [t for t in traps if t is not None]
    return bufs, (min(hit, key=lambda t: t[1]) if hit else None)


def bfs_full(row: np.ndarray, col: np.ndarray, nv: int, source: int = 0) -> tuple[np.ndarray, int]:
    L = lib()
    lvl = np.empty(nv, np.int32)
    r = np.ascontiguousarray(row, np.int32)
    c = np.ascontiguousarray(col, np.int32)
    levels = L.or_bfs_full(_ptr(r), _ptr(c), C.c_longlong(c.size), C.c_int(nv), C.c_int(source), _ptr(lvl))
    return lvl, levels


def hotspot_iterate(temp: np.ndarray, power: np.ndarray, rows: int, cols: int, params: dict,
                    iterations: int, bx: int = 16, by: int = 16, nthreads: int = 1) -> np.ndarray:
    """`iterations` ping-pong launches of hotspot.kn; returns the final grid."""
    L = lib()
    L.or_set_range(C.c_longlong(0), C.c_longlong(-1))
    a = np.ascontiguousarray(temp, np.float32).copy()
    b = np.zeros_like(a)
    p = np.ascontiguousarray(power, np.float32)
    g = Geom(-(-cols // bx), -(-rows // by), 1, bx, by, 1)
    t = OTrap()
    for _ in range(iterations):
        L.or_hotspot(g, _ptr(a), C.c_longlong(a.size), _ptr(p), C.c_longlong(p.size), _ptr(b),
                     C.c_longlong(b.size), C.c_int(rows), C.c_int(cols), C.c_double(params["sdc"]),
                     C.c_double(params["rx1"]), C.c_double(params["ry1"]), C.c_double(params["rz1"]),
                     C.c_double(params["amb"]), C.c_int(nthreads), C.byref(t))
        if t.kind:
            raise RuntimeError(f"oracle hotspot trapped: {t.kind} at block {t.block}")
        a, b = b, a
    return a


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
