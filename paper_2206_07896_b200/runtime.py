"""Runtime — the reference's launch runtime (runtime.py:1-350) on B200.

Same host API as `blockfuse.runtime`: `Runtime(arena, pool_size, policy,
hold_blocks, block_delay, seed)` with `.launch(routine, grid, block,
shmem_bytes, packed) -> KernelTask`, `.device_synchronize()`,
`.hold_new_blocks()`, `.shutdown()`, `.counters`, context manager; the fetch
policies and `resolve_grain`; `TaskQueue`; `KernelTask`; `RuntimeCounters`;
`PoolShutdown`; `RuntimeFault`.

What runs where: the queue, fetch loop, grain law and counters live in
libbfgpu.so (C++); every fetched block range is one grid launch of the
kernel's hand-written sm_100a implementation on a worker stream.  A pool
worker is an in-order CUDA stream on the arena's device (pool_size defaults
to 1: one stream already spreads a range over all 148 SMs; larger pools keep
the reference's fetch accounting and overlap independent launches).
"""

from __future__ import annotations

import ctypes as C
import logging
import struct
import threading
import weakref
from dataclasses import dataclass, field
from typing import Optional, Union

from . import _lib, routines
from ._lib import BfError, check
from .arena import DeviceArena, Trap

log = logging.getLogger(__name__)


class PoolShutdown(Exception):
    pass


class RuntimeFault(Exception):
    """An executor trap surfaced at synchronize, carrying the block id
    (runtime.py:32-38)."""

    def __init__(self, trap: Trap, block_id: int):
        self.trap = trap
        self.block_id = block_id
        super().__init__(f"block {block_id}: {trap}")


# ---------------------------------------------------------------------------
# geometry and packed arguments (syntax.py:31-71, executor.py:42-75,
# hostprog.py:390-414)
# ---------------------------------------------------------------------------

@dataclass
class Dim3:
    x: int = 1
    y: int = 1
    z: int = 1

    def __post_init__(self):
        if min(self.x, self.y, self.z) < 1:
            raise ValueError(f"dim3 components must be >= 1, got {self}")
        if self.x * self.y * self.z > 2**31 - 1:
            raise ValueError(f"dim3 product overflows i32: {self}")

    @property
    def total(self) -> int:
        return self.x * self.y * self.z

    def axis(self, axis: str) -> int:
        return getattr(self, axis)


def delinearize(i: int, dim) -> tuple[int, int, int]:
    return i % dim.x, (i // dim.x) % dim.y, i // (dim.x * dim.y)


def linearize(x: int, y: int, z: int, dim) -> int:
    return ((z * dim.y) + y) * dim.x + x


@dataclass
class ArgSlot:
    kind: str  # "i32" | "i64" | "f32" | "f64" | "handle"
    value: Union[int, float]


@dataclass
class PackedArgs:
    slots: list


_SLOT_FMT = {"i32": (struct.Struct("<iii4x"), 0), "i64": (struct.Struct("<iiq"), 1),
             "f32": (struct.Struct("<iid"), 2), "f64": (struct.Struct("<iid"), 3),
             "handle": (struct.Struct("<iiI4x"), 4)}


def pack_slots(packed) -> tuple[C.Array, int]:
    """Reference PackedArgs (or any object with .slots of (kind, value)) ->
    contiguous bf_slot array (16 B per slot).  f32 slots keep the unrounded
    double.  The packed array is cached on the PackedArgs object and reused
    while every slot is the same object holding the same kind and value
    objects (slots are mutable; the cache keeps the value objects alive, so
    identity implies the same value — 0.0 and -0.0 are different objects),
    which takes the packing off the launch path of host loops that relaunch
    the same arguments (hotspot's ping-pong, the BFS level loop)."""
    slots = packed.slots if packed is not None else ()
    cached = getattr(packed, "_bf_packed", None)
    if cached is not None and len(cached[0]) == len(slots):
        for (so, k, v), s in zip(cached[0], slots):
            if s is not so or s.kind is not k or s.value is not v:
                break
        else:
            return cached[1], cached[2]
    arr, n = _pack_slots(slots)
    try:
        packed._bf_packed = ([(s, s.kind, s.value) for s in slots], arr, n)
    except AttributeError:  # __slots__ objects (or no .kind/.value): no cache
        pass
    return arr, n


def _pack_slots(slots) -> tuple[C.Array, int]:
    n = len(slots)
    buf = bytearray(16 * max(n, 1))
    i = -1
    for s in slots:
        i += 1
        kind = s.kind
        ent = _SLOT_FMT.get(kind)
        if ent is None:
            raise Trap("TypeFault", f"unknown slot kind {kind!r}")
        fmt, code = ent
        v = float(s.value) if code in (2, 3) else int(s.value)
        if code == 0:
            v = (v + 2**31) % 2**32 - 2**31  # i32 slot: two's complement like ctypes
        elif code == 4:
            v &= 0xFFFFFFFF
        fmt.pack_into(buf, 16 * i, code, 0, v)
    t = _SLOT_ARRAYS.get(n)
    if t is None:
        t = _SLOT_ARRAYS[n] = _lib.Slot * max(n, 1)
    return t.from_buffer(buf), n


_SLOT_ARRAYS: dict = {}


# ---------------------------------------------------------------------------
# fetch policies (runtime.py:45-101)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Average:
    pass


@dataclass(frozen=True)
class Fixed:
    grain: int

    def __post_init__(self):
        if self.grain < 1:
            raise ValueError(f"grain must be >= 1, got {self.grain}")


@dataclass(frozen=True)
class AutoAggressive:
    light_kernel_threshold: int = 64


FetchPolicy = Union[Average, Fixed, AutoAggressive]


def parse_policy(text: str) -> FetchPolicy:
    if text == "average":
        return Average()
    if text == "auto":
        return AutoAggressive()
    if text.startswith("fixed:"):
        return Fixed(int(text[len("fixed:"):]))
    raise ValueError(f"unknown policy {text!r} (want average | fixed:<g> | auto)")


def resolve_grain(policy: FetchPolicy, grid_size: int, pool_size: int,
                  kernel_stats=None) -> int:
    """Blocks claimed per fetch for one launch (native bf_resolve_grain)."""
    if grid_size < 1 or pool_size < 1:
        raise ValueError("grid_size and pool_size must be >= 1")
    # duck-typed so the reference's own policy objects work too
    kind = type(policy).__name__
    if kind == "Average" and kernel_stats is not None:
        # hot path: ceil(G/P) (runtime.py:83), identical to the native law
        return -(-grid_size // pool_size)
    if kind == "Average":
        code, fixed, thr = _lib.POLICY_AVERAGE, 0, 0
    elif kind == "Fixed":
        code, fixed, thr = _lib.POLICY_FIXED, int(policy.grain), 0
    elif kind == "AutoAggressive":
        code, fixed, thr = _lib.POLICY_AUTO, 0, int(policy.light_kernel_threshold)
    else:
        raise ValueError(f"unknown fetch policy {policy!r}")
    atomics, est = -1, -1
    if kernel_stats is not None:
        atomics = 1 if kernel_stats.has_atomics() else 0
        est = int(kernel_stats.static_instruction_estimate())
    g = C.c_int64()
    check(_lib.lib().bf_resolve_grain(code, fixed, grid_size, pool_size, atomics, est, thr,
                                      C.byref(g)))
    log.debug("resolve_grain(%s, grid=%d, pool=%d) -> %d", type(policy).__name__, grid_size,
              pool_size, g.value)
    return g.value


# ---------------------------------------------------------------------------
# tasks and counters (runtime.py:108-143)
# ---------------------------------------------------------------------------

class KernelTask:
    """A launched kernel's record: the paper's kernel struct plus the
    instrumentation `remaining`, `fetches`, `executed` (runtime.py:108-125).

    Constructed standalone (dummy tasks for TaskQueue tests) it is a plain
    record; returned by Runtime.launch it reads the live native task."""

    def __init__(self, routine, args, gridDim, blockDim, dynamic_shared_mem_size: int,
                 totalBlocks: int, block_per_fetch: int, curr_blockId: int = 0):
        self.routine = routine
        self.args = args
        self.gridDim = gridDim
        self.blockDim = blockDim
        self.dynamic_shared_mem_size = dynamic_shared_mem_size
        self.totalBlocks = totalBlocks
        self.block_per_fetch = block_per_fetch
        self._curr = curr_blockId
        self._fetches = 0
        self._remaining = totalBlocks
        self._executed: Optional[list] = None
        self._rt: Optional["Runtime"] = None
        self._id = 0

    def _info(self):
        rt = self._rt
        if rt is None or not rt._native:
            return None
        info = _lib.TaskInfo()
        check(_lib.lib().bf_task_get(rt._native, self._id, C.byref(info)))
        return info

    @property
    def curr_blockId(self) -> int:
        i = self._info()
        if i is not None:
            self._curr = i.curr_block_id
        return self._curr

    @curr_blockId.setter
    def curr_blockId(self, v: int) -> None:
        self._curr = v

    @property
    def fetches(self) -> int:
        i = self._info()
        if i is not None:
            self._fetches = i.fetches
        return self._fetches

    @fetches.setter
    def fetches(self, v: int) -> None:
        self._fetches = v

    @property
    def remaining(self) -> int:
        i = self._info()
        if i is not None:
            self._remaining = i.remaining
        return self._remaining

    @remaining.setter
    def remaining(self, v: int) -> None:
        self._remaining = v

    @property
    def executed(self) -> list:
        rt = self._rt
        if rt is not None and rt._native:
            buf = (C.c_int32 * max(self.totalBlocks, 1))()
            check(_lib.lib().bf_task_executed(rt._native, self._id, buf, self.totalBlocks))
            self._executed = list(buf)[: self.totalBlocks]
        if self._executed is None:
            self._executed = [0] * self.totalBlocks
        return self._executed

    def __repr__(self) -> str:
        name = getattr(self.routine, "name", "?")
        return (f"KernelTask({name}, grid={self.gridDim}, block={self.blockDim}, "
                f"total={self.totalBlocks}, grain={self.block_per_fetch})")


@dataclass
class RuntimeCounters:
    fetch_count: int = 0
    blocks_executed: int = 0
    busy_blocks: list = field(default_factory=list)  # per worker
    syncs: int = 0
    queue_waits: int = 0

    def to_dict(self) -> dict:
        return {
            "blocks_executed": self.blocks_executed,
            "busy_blocks": list(self.busy_blocks),
            "fetch_count": self.fetch_count,
            "queue_waits": self.queue_waits,
            "syncs": self.syncs,
        }


class TaskQueue:
    """FIFO of tasks with the reference's fetch protocol (runtime.py:146-205),
    backed by the native queue the runtime's dispatcher uses."""

    def __init__(self, counters: RuntimeCounters):
        self._q = C.c_void_p()
        check(_lib.lib().bf_queue_create(C.byref(self._q)))
        self._cv = threading.Condition()
        self._tasks: dict[int, KernelTask] = {}
        self._next = 1
        self._closed = False
        self._counters = counters

    def __del__(self):
        try:
            if self._q:
                _lib.lib().bf_queue_destroy(self._q)
        except Exception:
            pass

    def held_by_me(self) -> bool:
        # the native guard is never held between calls
        return False

    def push(self, task: KernelTask) -> None:
        with self._cv:
            tag = self._next
            self._next += 1
            rc = _lib.lib().bf_queue_push(self._q, tag, task.totalBlocks, task.block_per_fetch)
            if rc == _lib.E_SHUTDOWN:
                raise PoolShutdown("launch after shutdown")
            check(rc)
            self._tasks[tag] = task
            self._cv.notify_all()

    def close(self) -> None:
        with self._cv:
            self._closed = True
            check(_lib.lib().bf_queue_close(self._q))
            self._cv.notify_all()

    def fetch(self):
        with self._cv:
            while True:
                got = C.c_int32()
                tag = C.c_uint64()
                first = C.c_int64()
                count = C.c_int64()
                check(_lib.lib().bf_queue_fetch(self._q, C.byref(got), C.byref(tag),
                                                C.byref(first), C.byref(count)))
                if got.value:
                    break
                if self._closed:
                    return None
                self._counters.queue_waits += 1
                self._cv.wait()
            task = self._tasks[tag.value]
            task.curr_blockId = first.value + count.value
            task.fetches = task.fetches + 1
            self._counters.fetch_count += 1
            if task.curr_blockId == task.totalBlocks:
                del self._tasks[tag.value]
            return task, first.value, count.value

    def is_empty(self) -> bool:
        e = C.c_int32()
        check(_lib.lib().bf_queue_is_empty(self._q, C.byref(e)))
        return bool(e.value)


# ---------------------------------------------------------------------------
# the runtime
# ---------------------------------------------------------------------------

def default_pool_size() -> int:
    return 1


class Runtime:
    """Worker pool (CUDA streams) plus task queue; created and joined once.

    `hold_blocks=True` gates all block execution until the next
    device_synchronize; `block_delay` inserts a random device-side sleep of up
    to that many seconds before each fetched range (seeded).  `instrument=True`
    makes every launch count per-block executions on the device.
    `fetch="device"` moves block fetching onto the GPU: a launch of a kernel
    that supports it is one persistent grid whose CTAs claim
    block_per_fetch blocks at a time from a device counter (the reference's
    worker fetch loop, runtime.py:175-201, 305-350); "host" (default) issues
    every fetched range as its own grid launch."""

    def __init__(self, arena: DeviceArena, pool_size: Optional[int] = None,
                 policy: FetchPolicy = Average(), hold_blocks: bool = False,
                 block_delay: float = 0.0, seed: int = 0, instrument: bool = False,
                 fetch: str = "host"):
        if fetch not in ("host", "device"):
            raise ValueError(f"fetch must be 'host' or 'device', got {fetch!r}")
        self.arena = arena
        self.pool_size = pool_size if pool_size is not None else default_pool_size()
        if self.pool_size < 1:
            raise ValueError(f"pool size must be >= 1, got {self.pool_size}")
        self.policy = policy
        self._native = C.c_void_p()
        flags = (_lib.FLAG_HOLD_BLOCKS if hold_blocks else 0) | \
                (_lib.FLAG_INSTRUMENT if instrument else 0) | \
                (_lib.FLAG_DEVICE_FETCH if fetch == "device" else 0)
        self.fetch = fetch
        check(_lib.lib().bf_runtime_create(arena.native, self.pool_size, flags, float(block_delay),
                                           seed & (2**64 - 1), C.byref(self._native)))
        # weak: a task keeps its runtime alive (it reads the native record),
        # the runtime must not keep its tasks alive (no reference cycle, so
        # runtime -> arena teardown order stays refcount-driven)
        self._tasks: list = []  # weakref.ref per launched task (pruned as it grows)
        self._tasks_prune_at = 1024
        self._shut_down = False
        # reusable launch scratch (the reference is driven by one host thread)
        self._tid = C.c_uint64()
        self._tid_addr = C.addressof(self._tid)
        # routine -> (routine, encoded registry key, warp size, fingerprint), by
        # identity: resolve (fingerprinting a reference MpmdKernel) runs once
        self._rcache: dict = {}
        self._bf_launch_desc = _lib.lib().bf_launch_described

    # -- host API ---------------------------------------------------------------
    def launch(self, routine, grid, block, shmem_bytes: int, packed) -> KernelTask:
        """Enqueue a kernel; returns immediately, never waits for the device."""
        return self._launch(routine, grid, block, shmem_bytes, packed, None)

    def launch_range(self, routine, grid, block, shmem_bytes: int, packed, first: int,
                     count: int) -> KernelTask:
        """Enqueue only logical blocks [first, first+count) of the grid: one
        worker's share (multi-GPU ranks, parallel.py).  The task has `count`
        blocks; its executed[] is indexed from `first`."""
        return self._launch(routine, grid, block, shmem_bytes, packed, (first, count))

    def _resolved(self, routine):
        ent = self._rcache.get(id(routine))
        if ent is None or ent[0] is not routine or routines.FORCE_JIT:
            name, _, warp_size = routines.resolve(routine)
            fp = None
            if not name.startswith("jit:") and hasattr(routine, "to_dict"):
                fp = C.create_string_buffer(bytes.fromhex(routines.fingerprint_of(routine.to_dict())), 32)
            ent = (routine, name.encode(), warp_size, fp)
            if len(self._rcache) > 256:
                self._rcache.clear()
            self._rcache[id(routine)] = ent  # holds the routine: its id stays unique
        return ent

    def _launch(self, routine, grid, block, shmem_bytes, packed, rng) -> KernelTask:
        if self._shut_down:
            raise PoolShutdown("launch after shutdown")
        ent = self._resolved(routine)
        total = grid.x * grid.y * grid.z if rng is None else rng[1]
        if self.policy.__class__.__name__ == "Average":
            if total < 1:
                raise ValueError("grid_size and pool_size must be >= 1")
            grain = -(-total // self.pool_size)  # runtime.py:83, the native law's hot path
        else:
            grain = resolve_grain(self.policy, total, self.pool_size, routine)
        task = KernelTask(routine, packed, grid, block, shmem_bytes, totalBlocks=total,
                          block_per_fetch=grain)
        slots, n = pack_slots(packed)
        # one cached launch descriptor per (routine, geometry, grain, range) on
        # the PackedArgs: a single pointer crosses ctypes per launch
        dkey = (ent[1], grid.x, grid.y, grid.z, block.x, block.y, block.z, shmem_bytes, grain, rng)
        cached = getattr(packed, "_bf_desc", None)
        if cached is not None and cached[0] == dkey and cached[2] is slots:
            d = cached[1]
        else:
            d = _lib.LaunchDesc()
            d.kernel = ent[1]
            d.fingerprint = C.addressof(ent[3]) if ent[3] is not None else None
            d.grid[0], d.grid[1], d.grid[2] = grid.x, grid.y, grid.z
            d.block[0], d.block[1], d.block[2] = block.x, block.y, block.z
            d.shmem_bytes = int(shmem_bytes)
            d.slots = C.addressof(slots)
            d.nslots = n
            d.warp_size = ent[2]
            d.first, d.count = (0, -1) if rng is None else (int(rng[0]), int(rng[1]))
            d.grain = grain
            try:
                packed._bf_desc = (dkey, d, slots, ent)  # keeps the slots and fingerprint alive
            except AttributeError:
                self._last_desc = (d, slots, ent)
        rc = self._bf_launch_desc(self._native, C.addressof(d), self._tid_addr)
        if rc == _lib.E_SHUTDOWN:
            raise PoolShutdown("launch after shutdown")
        if rc == _lib.E_UNKNOWN_KERNEL:
            raise routines.KernelNotImplemented(_lib.last_error())
        check(rc)
        task._rt = self
        task._id = self._tid.value
        self._tasks.append(weakref.ref(task))
        if len(self._tasks) > self._tasks_prune_at:
            self._tasks = [r for r in self._tasks if r() is not None]
            self._tasks_prune_at = max(1024, 2 * len(self._tasks))
        return task

    def device_synchronize(self) -> None:
        """Return once every fetched range finished; re-raise the first trap."""
        fault = _lib.Fault()
        rc = _lib.lib().bf_synchronize(self._native, C.byref(fault))
        if rc == _lib.E_FAULT:
            kind = _lib.TRAP_NAMES.get(fault.kind, "TypeFault")
            trap = Trap(kind, fault.message.decode(errors="replace"),
                        kernel=fault.kernel.decode(errors="replace"))
            raise RuntimeFault(trap, fault.block_id)
        check(rc)

    def unfinished_tasks(self) -> list:
        live = [r() for r in self._tasks]
        return sorted((t for t in live if t is not None and t.remaining > 0), key=lambda t: t._id)

    def hold_new_blocks(self) -> None:
        check(_lib.lib().bf_hold_new_blocks(self._native))

    def worker_stream(self, worker: int = 0) -> int:
        """cudaStream_t of a worker, as an int (for torch.cuda.ExternalStream)."""
        s = C.c_void_p()
        check(_lib.lib().bf_worker_stream(self._native, worker, C.byref(s)))
        return s.value or 0

    @property
    def counters(self) -> RuntimeCounters:
        c = _lib.Counters()
        busy = (C.c_int64 * self.pool_size)()
        check(_lib.lib().bf_counters_get(self._native, C.byref(c), busy, self.pool_size))
        return RuntimeCounters(c.fetch_count, c.blocks_executed, list(busy), c.syncs,
                               c.queue_waits)

    def shutdown(self) -> None:
        """Idempotent; drains the device.  The native record stays alive (tasks
        and counters remain readable) until this object is collected."""
        if self._shut_down:
            return
        self._shut_down = True
        check(_lib.lib().bf_shutdown(self._native))

    def __enter__(self) -> "Runtime":
        return self

    def __exit__(self, *exc) -> None:
        self.shutdown()

    def __del__(self):
        try:
            if self._native:
                _lib.lib().bf_runtime_destroy(self._native)
                self._native = C.c_void_p()
        except Exception:
            pass
