"""Runtime tests, mirroring the reference's tests/test_runtime.py and the
runtime criteria of tests/test_acceptance.py (fetch protocol, grain law,
scheduling, exactly-once, traps, adversarial schedules) against this
package's native runtime.  Queue and grain tests need no GPU."""

import random

import numpy as np

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import instances as I
from conftest import has_gpu
from gpu_helpers import bit_equal, gpu_run, materialize
from paper_2206_07896_b200 import (ArgSlot, AutoAggressive, Average, DeviceArena, Dim3, Fixed,
                                   KernelTask, PackedArgs, PoolShutdown, Runtime, RuntimeCounters,
                                   RuntimeFault, TaskQueue, parse_policy, resolve_grain, routines)
import oracle


def _task(total, grain):
    return KernelTask(routines.get("vecadd"), None, Dim3(total), Dim3(1), 0,
                      totalBlocks=total, block_per_fetch=grain)


def _drain(queue):
    ranges = []
    while not queue.is_empty():
        task, first, count = queue.fetch()
        ranges.append((first, count))
    return ranges


class TestTaskQueue:  # test_runtime.py:48-111
    def test_even_split(self):
        q = TaskQueue(RuntimeCounters())
        q.push(_task(16, 4))
        assert _drain(q) == [(0, 4), (4, 4), (8, 4), (12, 4)]

    def test_ragged_tail(self):
        q = TaskQueue(RuntimeCounters())
        q.push(_task(10, 4))
        assert _drain(q) == [(0, 4), (4, 4), (8, 2)]

    def test_two_fetches(self):
        q = TaskQueue(RuntimeCounters())
        q.push(_task(12, 6))
        assert _drain(q) == [(0, 6), (6, 6)]

    def test_pop_happens_on_last_fetch(self):
        q = TaskQueue(RuntimeCounters())
        task = _task(8, 8)
        q.push(task)
        got, first, count = q.fetch()
        assert (got, first, count) == (task, 0, 8)
        assert q.is_empty()

    def test_fifo_across_tasks(self):
        q = TaskQueue(RuntimeCounters())
        a, b = _task(4, 2), _task(2, 2)
        q.push(a)
        q.push(b)
        order = [q.fetch()[0] for _ in range(3)]
        assert order == [a, a, b]

    def test_fetch_returns_none_after_close(self):
        q = TaskQueue(RuntimeCounters())
        q.close()
        assert q.fetch() is None

    def test_push_after_close_raises(self):
        q = TaskQueue(RuntimeCounters())
        q.close()
        with pytest.raises(PoolShutdown):
            q.push(_task(1, 1))

    def test_guard_not_held_outside_calls(self):
        q = TaskQueue(RuntimeCounters())
        q.push(_task(1, 1))
        assert not q.held_by_me()
        q.fetch()
        assert not q.held_by_me()

    def test_fetch_blocks_until_push(self):
        import threading
        q = TaskQueue(RuntimeCounters())
        got = []
        t = threading.Thread(target=lambda: got.append(q.fetch()))
        t.start()
        task = _task(3, 3)
        q.push(task)
        t.join(timeout=10)
        assert got and got[0][0] is task

    @settings(max_examples=100, deadline=None)
    @given(total=st.integers(1, 300), grain=st.integers(1, 300))
    def test_fetch_count_is_ceil_total_over_grain(self, total, grain):
        counters = RuntimeCounters()
        q = TaskQueue(counters)
        task = _task(total, min(grain, total))
        q.push(task)
        ranges = _drain(q)
        assert len(ranges) == -(-total // min(grain, total))
        assert counters.fetch_count == len(ranges) == task.fetches
        covered = [b for first, count in ranges for b in range(first, first + count)]
        assert covered == list(range(total))


class TestGrainResolution:  # test_runtime.py:114-147
    def test_average_is_ceil(self):
        assert resolve_grain(Average(), 12, 3) == 4
        assert resolve_grain(Average(), 13, 3) == 5
        assert resolve_grain(Average(), 2, 8) == 1

    def test_fixed_clamped_to_grid(self):
        assert resolve_grain(Fixed(6), 100, 4) == 6
        assert resolve_grain(Fixed(500), 100, 4) == 100

    def test_fixed_rejects_nonpositive(self):
        with pytest.raises(ValueError):
            Fixed(0)

    def test_auto_doubles_for_atomic_kernels(self):
        hist = routines.get("hist")
        assert hist.has_atomics()
        assert resolve_grain(AutoAggressive(), 12, 3, hist) == 8
        assert resolve_grain(AutoAggressive(), 6, 3, hist) == 4

    def test_auto_widens_light_kernels(self):
        vec = routines.get("vecadd")
        assert vec.static_instruction_estimate() < 64
        assert resolve_grain(AutoAggressive(), 12, 3, vec) == 6

    def test_auto_without_stats_matches_average(self):
        assert resolve_grain(AutoAggressive(), 12, 3) == 4

    def test_parse_policy(self):
        assert parse_policy("average") == Average()
        assert parse_policy("auto") == AutoAggressive()
        assert parse_policy("fixed:7") == Fixed(7)
        with pytest.raises(ValueError):
            parse_policy("eager")

    def test_invalid_sizes(self):
        with pytest.raises(ValueError):
            resolve_grain(Average(), 0, 3)
        with pytest.raises(ValueError):
            resolve_grain(Average(), 3, 0)


def test_fetch_count_law():  # test_acceptance.py:120-151
    rng = random.Random(7)
    for _ in range(200):
        total = rng.randint(1, 500)
        grain = rng.randint(1, total)
        q = TaskQueue(RuntimeCounters())
        task = _task(total, grain)
        q.push(task)
        while not q.is_empty():
            q.fetch()
        assert task.fetches == -(-total // grain)
        assert task.curr_blockId == total
    grain = resolve_grain(Average(), 12, 3)
    assert grain == 4
    q = TaskQueue(RuntimeCounters())
    task = _task(12, grain)
    q.push(task)
    while not q.is_empty():
        q.fetch()
    assert task.fetches == 3


def test_average_policy_exhaustive():  # test_acceptance.py:156-168
    for grid in range(1, 65):
        for pool in range(1, 65):
            grain = resolve_grain(Average(), grid, pool)
            assert grain == -(-grid // pool)
            assert -(-grid // grain) <= pool


# ---------------------------------------------------------------------------
# scheduling on the device
# ---------------------------------------------------------------------------

gpu = pytest.mark.gpu


@pytest.fixture
def need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")


def _hist_instance():
    return I.hist(random.Random(5))


@gpu
@pytest.mark.parametrize("pool", [1, 2, 4])
@pytest.mark.parametrize("grain", [1, 3, "average"])
def test_every_block_runs_exactly_once(need_gpu, pool, grain):  # test_runtime.py:155-165
    inst = _hist_instance()
    policy = Average() if grain == "average" else Fixed(grain)
    outs, trap, task, counters = gpu_run(inst, pool_size=pool, policy=policy, instrument=True)
    assert trap is None
    assert task.executed == [1] * inst.grid.total
    assert counters.blocks_executed == inst.grid.total
    want, _ = oracle.run(inst)
    assert bit_equal(outs["counts"], want["counts"])


@gpu
def test_launch_does_not_wait_for_workers(need_gpu):  # test_runtime.py:167-178
    inst = _hist_instance()
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    with Runtime(arena, pool_size=2, hold_blocks=True) as rt:
        task = rt.launch(routines.get("hist"), Dim3(inst.grid.x), Dim3(inst.block.x), 0, packed)
        # gated: launch returned with all blocks still pending
        assert task.remaining == inst.grid.total
        assert rt.unfinished_tasks() == [task]
        assert arena.to_list(handles["counts"]) == [0] * len(inst.buffer("counts").values)
        rt.device_synchronize()
        assert task.remaining == 0
        assert rt.unfinished_tasks() == []
    want, _ = oracle.run(inst)
    assert bit_equal(arena.to_numpy(handles["counts"]), want["counts"])


@gpu
def test_remaining_falls_without_synchronize(need_gpu):
    """task.remaining reaches 0 by polling alone (no device_synchronize), as a
    host spinning on the reference's counters would: completion is tracked
    lazily by an event that covers every fetch issued before the query."""
    import time
    inst = I.vecadd(random.Random(12))
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    with Runtime(arena, pool_size=2) as rt:
        tasks = [rt.launch(routines.get("vecadd"), Dim3(inst.grid.x), Dim3(inst.block.x), 0, packed)
                 for _ in range(5)]
        deadline = time.time() + 30
        while any(t.remaining for t in tasks) and time.time() < deadline:
            time.sleep(0.001)
        assert [t.remaining for t in tasks] == [0] * 5
        assert rt.unfinished_tasks() == []
        assert rt.counters.blocks_executed == 5 * inst.grid.total


@gpu
def test_hold_new_blocks_rearms_the_gate(need_gpu):
    inst = I.vecadd(random.Random(11))
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    with Runtime(arena, pool_size=2) as rt:
        rt.hold_new_blocks()
        task = rt.launch(routines.get("vecadd"), Dim3(inst.grid.x), Dim3(inst.block.x), 0, packed)
        assert task.remaining == inst.grid.total
        rt.device_synchronize()
        assert task.remaining == 0


@gpu
def test_worker_busy_counts_sum_to_blocks(need_gpu):  # test_runtime.py:180-185
    inst = I.vecadd(random.Random(11))
    _, _, _, counters = gpu_run(inst, pool_size=4, policy=Fixed(1))
    assert sum(counters.busy_blocks) == inst.grid.total
    assert len(counters.busy_blocks) == 4
    assert counters.fetch_count == inst.grid.total


@gpu
def test_launch_after_shutdown_raises(need_gpu):  # test_runtime.py:197-201
    rt = Runtime(DeviceArena(), pool_size=1)
    rt.shutdown()
    with pytest.raises(PoolShutdown):
        rt.launch(routines.get("vecadd"), Dim3(1), Dim3(1), 0, None)


@gpu
def test_shutdown_is_idempotent(need_gpu):
    rt = Runtime(DeviceArena(), pool_size=2)
    rt.shutdown()
    rt.shutdown()


@gpu
def test_trap_surfaces_as_runtime_fault(need_gpu):  # test_runtime.py:210-225
    arena = DeviceArena()
    h = arena.alloc("f32", 4)
    with Runtime(arena, pool_size=2) as rt:
        rt.launch(routines.get("vecadd"), Dim3(4), Dim3(4), 0,
                  PackedArgs([ArgSlot("handle", h)] * 3 + [ArgSlot("i32", 16)]))
        with pytest.raises(RuntimeFault) as e:
            rt.device_synchronize()
        assert e.value.trap.kind == "OutOfBounds"
        assert e.value.block_id == 1  # ids 4..7 are the first out of range
        # the reference keeps the first fault: later syncs re-raise it
        with pytest.raises(RuntimeFault):
            rt.device_synchronize()


@gpu
def test_wrong_slot_kind_is_a_type_fault(need_gpu):
    arena = DeviceArena()
    h = arena.alloc("f32", 4)
    with Runtime(arena) as rt:
        rt.launch(routines.get("vecadd"), Dim3(1), Dim3(4), 0,
                  PackedArgs([ArgSlot("handle", h)] * 3 + [ArgSlot("f32", 4.0)]))
        with pytest.raises(RuntimeFault) as e:
            rt.device_synchronize()
        assert e.value.trap.kind == "TypeFault"


@gpu
def test_dangling_handle_is_out_of_bounds(need_gpu):
    arena = DeviceArena()
    h = arena.alloc("f32", 4)
    arena.free(h)
    with Runtime(arena) as rt:
        rt.launch(routines.get("vecadd"), Dim3(1), Dim3(4), 0,
                  PackedArgs([ArgSlot("handle", h)] * 3 + [ArgSlot("i32", 4)]))
        with pytest.raises(RuntimeFault) as e:
            rt.device_synchronize()
        assert e.value.trap.kind == "OutOfBounds"


@gpu
def test_device_detected_trap(need_gpu):
    inst = I.hist(random.Random(3))
    inst.buffers[0].values[5] = -7  # negative bin -> OutOfBounds on the device
    inst.args[2] = ("i32", max(inst.args[2][1], 6))
    _, trap, _, _ = gpu_run(inst)
    assert trap is not None and trap[0] == "OutOfBounds"


@gpu
def test_block_delay_preserves_results(need_gpu):  # test_runtime.py:227-238
    inst = I.hist(random.Random(17))
    outs, trap, _, _ = gpu_run(inst, pool_size=4, policy=Fixed(2))
    want, _ = oracle.run(inst)
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    with Runtime(arena, pool_size=4, policy=Fixed(2), block_delay=0.001, seed=2) as rt:
        rt.launch(routines.get("hist"), Dim3(inst.grid.x), Dim3(inst.block.x), 0, packed)
        rt.device_synchronize()
    assert bit_equal(arena.to_numpy(handles["counts"]), want["counts"])


@gpu
def test_concurrent_launches_from_many_host_calls(need_gpu):  # test_runtime.py:240-253
    inst = I.vecadd(random.Random(11))
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    with Runtime(arena, pool_size=4) as rt:
        tasks = [rt.launch(routines.get("vecadd"), Dim3(inst.grid.x), Dim3(inst.block.x), 0, packed)
                 for _ in range(5)]
        rt.device_synchronize()
    assert all(t.remaining == 0 for t in tasks)
    want, _ = oracle.run(inst)
    assert bit_equal(arena.to_numpy(handles["c"]), want["c"])


@gpu
def test_exactly_once_histogram(need_gpu):  # test_acceptance.py:273-290
    inst = I.hist(random.Random(4))
    want, _ = oracle.run(inst)
    total = inst.grid.total
    for pool in (1, 2, 4, 8):
        for grain in (Fixed(1), Average(), Fixed(total)):
            outs, trap, task, _ = gpu_run(inst, pool_size=pool, policy=grain, instrument=True)
            assert trap is None
            assert task.executed == [1] * total
            assert bit_equal(outs["counts"], want["counts"])


@gpu
def test_warp_mode(need_gpu):  # test_acceptance.py:295-322
    rng = random.Random(13)
    for _ in range(10):
        inst = I.wreduce(rng)
        inst.block = I.Geom(64)
        inst.grid = I.Geom(4)
        outs, trap, _, _ = gpu_run(inst, pool_size=2)
        want, _ = oracle.run(inst)
        assert trap is None and bit_equal(outs["out"], want["out"])


@gpu
def test_unknown_kernel_is_rejected(need_gpu):
    arena = DeviceArena()

    class Foreign:
        name = "writer"
    with Runtime(arena) as rt:
        with pytest.raises(routines.KernelNotImplemented):
            rt.launch(Foreign(), Dim3(1), Dim3(1), 0, PackedArgs([]))


@gpu
def test_arena_surface(need_gpu):  # arena.py:75-152
    from paper_2206_07896_b200 import Trap
    a = DeviceArena()
    h1 = a.alloc("i32", 20)
    h2 = a.alloc("f64", 1)
    assert (h1, h2) == (1, 2)
    assert a.base_address(h1) % 64 == 0 and a.base_address(h2) == 128
    assert a.to_list(h1) == [0] * 20
    a.fill(h1, range(25))
    assert a.to_list(h1) == list(range(20))
    hf = a.alloc("f32", 3)
    a.fill(hf, [0.1, 0.2])
    assert a.to_list(hf) == [I.f32(0.1), I.f32(0.2), 0.0]
    raw = a.to_bytes(h1)
    assert len(raw) == 80
    a.from_bytes(h1, bytes(80))
    assert a.to_list(h1) == [0] * 20
    with pytest.raises(ValueError):
        a.from_bytes(h1, bytes(4))
    with pytest.raises(Trap):
        a.read(h1, 20)
    a.write(h1, 3, 7)
    assert a.read(h1, 3) == 7
    a.free(h1)
    with pytest.raises(Trap):
        a.to_list(h1)
    assert a.alloc("i32", 0) == 4  # never reused
    with pytest.raises(ValueError):
        a.alloc("i32", -1)


def test_packed_cache_distinguishes_negative_zero():
    """the packed-slot cache must not reuse 0.0's packing for -0.0."""
    import struct

    from paper_2206_07896_b200 import ArgSlot, PackedArgs
    from paper_2206_07896_b200.runtime import pack_slots
    pk = PackedArgs([ArgSlot("f32", 0.0)])
    arr, n = pack_slots(pk)
    assert bytes(arr)[8:16] == struct.pack("<d", 0.0)
    pk.slots[0] = ArgSlot("f32", -0.0)
    arr, n = pack_slots(pk)
    assert bytes(arr)[8:16] == struct.pack("<d", -0.0)


@pytest.mark.gpu
def test_launch_described_checks_fingerprint():
    """The C ABI's descriptor launch runs a registered kernel when the body
    fingerprint matches and refuses a different body under the same name."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    import ctypes as C
    import json
    from pathlib import Path
    from paper_2206_07896_b200 import ArgSlot, DeviceArena, PackedArgs, Runtime, _lib
    from paper_2206_07896_b200.runtime import pack_slots
    fps = json.loads((Path(__file__).resolve().parents[1] / "paper_2206_07896_b200" / "fingerprints.json").read_text())
    arena = DeviceArena()
    n = 1000
    a, b, c = (arena.alloc("f32", n) for _ in range(3))
    arena.upload_numpy(a, np.arange(n, dtype=np.float32))
    arena.upload_numpy(b, np.ones(n, np.float32))
    slots, ns = pack_slots(PackedArgs([ArgSlot("handle", a), ArgSlot("handle", b), ArgSlot("handle", c),
                                       ArgSlot("i32", n)]))
    with Runtime(arena) as rt:
        good = C.create_string_buffer(bytes.fromhex(fps["vecadd"]), 32)
        bad = C.create_string_buffer(bytes(32), 32)
        tid = C.c_uint64()
        for fp, want in ((good, _lib.OK), (bad, _lib.E_UNKNOWN_KERNEL), (None, _lib.OK)):
            d = _lib.LaunchDesc()
            d.kernel = b"vecadd"
            d.fingerprint = C.addressof(fp) if fp is not None else None
            d.grid[:] = (4, 1, 1)
            d.block[:] = (256, 1, 1)
            d.slots, d.nslots, d.warp_size, d.first, d.count, d.grain = C.addressof(slots), ns, 0, 0, -1, 4
            assert _lib.lib().bf_launch_described(rt._native, C.addressof(d), C.addressof(tid)) == want
        rt.device_synchronize()
    assert np.array_equal(arena.to_numpy(c), np.arange(n, dtype=np.float32) + 1)
