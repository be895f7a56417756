"""ctypes binding of libbfgpu.so (include/bfgpu.h).

This module is the whole Python↔native boundary.  It fails loudly when the
library is missing: there is no CPU fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libbfgpu.so"

# status codes (enum bf_status)
OK, E_INVALID, E_SHUTDOWN, E_TYPEFAULT, E_UNKNOWN_KERNEL, E_CUDA, E_DANGLING, E_FAULT, E_UNSUPPORTED = range(9)

# scalars / slot kinds
SCALARS = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}
SCALAR_NAMES = {v: k for k, v in SCALARS.items()}
SLOT_KINDS = {"i32": 0, "i64": 1, "f32": 2, "f64": 3, "handle": 4}
SLOT_NAMES = {v: k for k, v in SLOT_KINDS.items()}
TRAP_NAMES = {0: None, 1: "OutOfBounds", 2: "DivByZero", 3: "TypeFault", 4: "NonUniformTrip"}

POLICY_AVERAGE, POLICY_FIXED, POLICY_AUTO = 0, 1, 2
FLAG_HOLD_BLOCKS = 0x1
FLAG_INSTRUMENT = 0x2
FLAG_DEVICE_FETCH = 0x4

EXPORTS = [
    "bf_abi_version", "bf_last_error", "bf_device_count",
    "bf_arena_create", "bf_arena_destroy", "bf_alloc", "bf_free", "bf_view", "bf_buffer_info",
    "bf_upload", "bf_download", "bf_fill32", "bf_copy",
    "bf_queue_create", "bf_queue_destroy", "bf_queue_push", "bf_queue_fetch",
    "bf_queue_close", "bf_queue_is_empty", "bf_queue_task", "bf_queue_counters",
    "bf_resolve_grain",
    "bf_runtime_create", "bf_shutdown", "bf_runtime_destroy", "bf_launch", "bf_launch_range", "bf_launch_described",
    "bf_kernel_set_fingerprint",
    "bf_synchronize", "bf_hold_new_blocks", "bf_task_get", "bf_task_executed",
    "bf_counters_get", "bf_worker_stream",
    "bf_kernel_count", "bf_kernel_info",
    "bf_bfs_levels", "bf_bfs_levels_do", "bf_bfs_transpose", "bf_hotspot_run", "bf_jit_register",
    "bf_bfs_shard_create", "bf_bfs_shard_destroy", "bf_bfs_shard_bitmap", "bf_bfs_shard_begin",
    "bf_bfs_shard_expand", "bf_bfs_shard_merge", "bf_bfs_shard_merge_slice", "bf_bfs_shard_compact", "bf_bfs_shard_finish",
    "bf_kmeans_update",
]


class _SlotValue(C.Union):
    _fields_ = [("i32", C.c_int32), ("i64", C.c_int64), ("f64", C.c_double), ("handle", C.c_uint32)]


class Slot(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("v", _SlotValue)]


class Fault(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("block_id", C.c_int64),
                ("task_id", C.c_uint64), ("kernel", C.c_char * 32), ("message", C.c_char * 160)]


class LaunchDesc(C.Structure):
    _fields_ = [("kernel", C.c_char_p), ("fingerprint", C.c_void_p), ("grid", C.c_int32 * 3),
                ("block", C.c_int32 * 3), ("shmem_bytes", C.c_int64), ("slots", C.c_void_p),
                ("nslots", C.c_int32), ("warp_size", C.c_int32), ("first", C.c_int64), ("count", C.c_int64),
                ("grain", C.c_int64)]


class TaskInfo(C.Structure):
    _fields_ = [("total_blocks", C.c_int64), ("block_per_fetch", C.c_int64),
                ("curr_block_id", C.c_int64), ("fetches", C.c_int64), ("remaining", C.c_int64)]


class Counters(C.Structure):
    _fields_ = [("fetch_count", C.c_int64), ("blocks_executed", C.c_int64), ("syncs", C.c_int64),
                ("queue_waits", C.c_int64), ("pool_size", C.c_int32), ("_pad", C.c_int32)]


class BfError(RuntimeError):
    """A native call failed; `.code` is the bf_status."""

    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"bfgpu status {code}: {message}")


_lib = None


def _declare(lib) -> None:
    P = C.c_void_p
    i32, i64, u32, u64, dbl = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
    I32P, I64P, U32P, U64P = (C.POINTER(i32), C.POINTER(i64), C.POINTER(u32), C.POINTER(u64))
    sig = {
        "bf_abi_version": (C.c_int, []),
        "bf_last_error": (C.c_char_p, []),
        "bf_device_count": (C.c_int, [I32P]),
        "bf_arena_create": (C.c_int, [i32, C.POINTER(P)]),
        "bf_arena_destroy": (C.c_int, [P]),
        "bf_alloc": (C.c_int, [P, i32, i64, U32P]),
        "bf_free": (C.c_int, [P, u32]),
        "bf_view": (C.c_int, [P, u32, i64, i64, C.POINTER(u32)]),
        "bf_buffer_info": (C.c_int, [P, u32, I32P, I64P, U64P]),
        "bf_upload": (C.c_int, [P, u32, P, i64, i64]),
        "bf_download": (C.c_int, [P, u32, P, i64, i64]),
        "bf_fill32": (C.c_int, [P, u32, u32, i64, i64]),
        "bf_copy": (C.c_int, [P, u32, i64, u32, i64, i64]),
        "bf_queue_create": (C.c_int, [C.POINTER(P)]),
        "bf_queue_destroy": (C.c_int, [P]),
        "bf_queue_push": (C.c_int, [P, u64, i64, i64]),
        "bf_queue_fetch": (C.c_int, [P, I32P, U64P, I64P, I64P]),
        "bf_queue_close": (C.c_int, [P]),
        "bf_queue_is_empty": (C.c_int, [P, I32P]),
        "bf_queue_task": (C.c_int, [P, u64, I64P, I64P]),
        "bf_queue_counters": (C.c_int, [P, I64P, I64P]),
        "bf_resolve_grain": (C.c_int, [i32, i64, i64, i64, i32, i64, i64, I64P]),
        "bf_runtime_create": (C.c_int, [P, i32, u32, dbl, u64, C.POINTER(P)]),
        "bf_shutdown": (C.c_int, [P]),
        "bf_runtime_destroy": (C.c_int, [P]),
        "bf_launch": (C.c_int, [P, C.c_char_p, I32P, I32P, i64, C.POINTER(Slot), i32, i32, i64, U64P]),
        "bf_launch_range": (C.c_int, [P, C.c_char_p, I32P, I32P, i64, C.POINTER(Slot), i32, i32, i64, i64,
                                      i64, U64P]),
        "bf_launch_described": (C.c_int, [P, P, P]),
        "bf_kernel_set_fingerprint": (C.c_int, [C.c_char_p, C.c_char_p]),
        "bf_synchronize": (C.c_int, [P, C.POINTER(Fault)]),
        "bf_hold_new_blocks": (C.c_int, [P]),
        "bf_task_get": (C.c_int, [P, u64, C.POINTER(TaskInfo)]),
        "bf_task_executed": (C.c_int, [P, u64, I32P, i64]),
        "bf_counters_get": (C.c_int, [P, C.POINTER(Counters), I64P, i32]),
        "bf_worker_stream": (C.c_int, [P, i32, C.POINTER(P)]),
        "bf_kernel_count": (C.c_int, [I32P]),
        "bf_bfs_levels": (C.c_int, [P, u32, u32, u32, i32, i32, I32P]),
        "bf_bfs_levels_do": (C.c_int, [P, u32, u32, u32, u32, u32, i32, i32, I32P]),
        "bf_bfs_transpose": (C.c_int, [P, u32, u32, i32, u32, u32]),
        "bf_bfs_shard_create": (C.c_int, [P, i32, C.POINTER(P)]),
        "bf_bfs_shard_destroy": (C.c_int, [P]),
        "bf_bfs_shard_bitmap": (C.c_int, [P, C.POINTER(P), I64P]),
        "bf_bfs_shard_begin": (C.c_int, [P, i32, i64, i64]),
        "bf_bfs_shard_expand": (C.c_int, [P, u32, u32]),
        "bf_bfs_shard_merge": (C.c_int, [P, P, i32]),
        "bf_bfs_shard_merge_slice": (C.c_int, [P, P, i32, i64, i64]),
        "bf_bfs_shard_compact": (C.c_int, [P, u32, I64P]),
        "bf_bfs_shard_finish": (C.c_int, [P, u32, I32P]),
        "bf_kmeans_update": (C.c_int, [P, u32, u32, u32, i32, i32, u32, u32, i64, i64, I64P]),
        "bf_hotspot_run": (C.c_int, [P, u32, u32, u32, i32, i32, C.POINTER(dbl), i32, i32]),
        "bf_jit_register": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, i32, I32P, I32P, i32]),
        "bf_kernel_info": (C.c_int, [i32, C.c_char_p, i32, I32P, I32P, I32P, i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Load libbfgpu.so once; raise if it was never built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2206_07896_b200.build` "
                "(there is no CPU fallback)")
        _lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | C.RTLD_GLOBAL)
        _declare(_lib)
        _register_fingerprints(_lib)
    return _lib


def _register_fingerprints(L) -> None:
    """Expected body fingerprints of the hand-written kernels -> the C ABI
    (bf_kernel_set_fingerprint), so bf_launch_desc checks them natively."""
    import json
    fp_file = Path(__file__).resolve().parent / "fingerprints.json"
    if not fp_file.exists():
        return
    for name, hexfp in json.loads(fp_file.read_text()).items():
        raw = bytes.fromhex(hexfp)
        if len(raw) == 32:
            L.bf_kernel_set_fingerprint(name.encode(), raw)  # unknown names: ignored


def last_error() -> str:
    return lib().bf_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc != OK:
        raise BfError(rc, last_error())


def kernels() -> dict[str, list[tuple[str, str]]]:
    """Registered kernels: name -> [(slot kind, element scalar or None)]."""
    L = lib()
    n = C.c_int32()
    check(L.bf_kernel_count(C.byref(n)))
    out = {}
    for i in range(n.value):
        name = C.create_string_buffer(64)
        npar = C.c_int32()
        kinds = (C.c_int32 * 32)()
        scal = (C.c_int32 * 32)()
        check(L.bf_kernel_info(i, name, 64, C.byref(npar), kinds, scal, 32))
        out[name.value.decode()] = [
            (SLOT_NAMES[kinds[j]], SCALAR_NAMES[scal[j]] if kinds[j] == 4 else None)
            for j in range(npar.value)]
    return out


def device_count() -> int:
    n = C.c_int32()
    rc = lib().bf_device_count(C.byref(n))
    return n.value if rc == OK else 0
