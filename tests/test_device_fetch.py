"""Device-side block fetching (Runtime(fetch="device"), BF_FLAG_DEVICE_FETCH):
the paper's block fetching done by the GPU's own CTAs — one persistent grid
per launch whose CTAs claim block_per_fetch logical blocks at a time from a
device claim counter (/root/reference/pkg/src/blockfuse/runtime.py:175-201,
305-350).  Results equal the oracle for every policy and
pool size, every block runs exactly once (device-counted executed[]), and the
fetch / busy counters come from the device and obey the reference's
fetch-count law (runtime.py:83)."""

import random
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))

import instances as I  # noqa: E402
import oracle  # noqa: E402
from gpu_helpers import bit_equal, gpu_run  # noqa: E402

from paper_2206_07896_b200 import (ArgSlot, Average, DeviceArena, Dim3, Fixed, PackedArgs,  # noqa: E402
                                   Runtime, RuntimeFault, routines)

gpu = pytest.mark.gpu


@pytest.fixture
def need_gpu():
    from conftest import has_gpu
    if not has_gpu():
        pytest.skip("no CUDA device")


def test_fetch_argument_is_checked():
    with pytest.raises(ValueError):
        Runtime(DeviceArena.__new__(DeviceArena), fetch="gpu")


def _vecadd(n, bx=256, seed=1):
    a = np.random.default_rng(seed).uniform(-1, 1, n).astype(np.float32)
    b = np.random.default_rng(seed + 1).uniform(-1, 1, n).astype(np.float32)
    gx = -(-n // bx)
    return I.Instance("vecadd", I.Geom(gx), I.Geom(bx), 0,
                      [I.Buf("a", "f32", n, a), I.Buf("b", "f32", n, b), I.Buf("c", "f32", n, np.zeros(n, np.float32))],
                      [("buf", "a"), ("buf", "b"), ("buf", "c"), ("i32", n)], ["c"])


def _hist(n, nbins, bx=256, seed=3):
    pix = np.random.default_rng(seed).integers(0, 1 << 20, n).astype(np.int32)
    gx = -(-n // bx)
    return I.Instance("hist", I.Geom(gx), I.Geom(bx), 0,
                      [I.Buf("pix", "i32", n, pix), I.Buf("counts", "i32", nbins, np.zeros(nbins, np.int32))],
                      [("buf", "pix"), ("buf", "counts"), ("i32", n), ("i32", nbins)], ["counts"])


POLICIES = [("average", None), ("fixed1", Fixed(1)), ("fixed3", Fixed(3)), ("fixed64", Fixed(64)),
            ("fixed_huge", Fixed(1 << 30))]


@gpu
@pytest.mark.parametrize("pool", [1, 3])
@pytest.mark.parametrize("pname,policy", POLICIES)
def test_device_fetch_matches_oracle_and_counts(need_gpu, pool, pname, policy):
    cases = [_vecadd(1 << 16), _vecadd(5000 * 4 + 12), _hist(1 << 16, 16), _hist(70000, 1000), _hist(4096, 9000)]
    for inst in cases:
        want, trap = oracle.run(inst)
        assert trap is None
        got, got_trap, task, counters = gpu_run(inst, pool_size=pool, policy=policy, instrument=True, fetch="device")
        assert got_trap is None
        for buf in inst.outputs:
            assert bit_equal(got[buf], want[buf]), (inst.kernel, buf, pname, pool)
        total = inst.grid.x
        grain = task.block_per_fetch
        nfetch = -(-total // grain)
        assert task.fetches == nfetch
        assert task.remaining == 0
        assert list(task.executed) == [1] * total  # counted by the CTAs that ran them
        assert counters.fetch_count == nfetch and counters.blocks_executed == total
        assert sum(counters.busy_blocks) == total and len(counters.busy_blocks) == pool


@gpu
def test_device_fetch_counters_accumulate_over_launches(need_gpu):
    inst = _vecadd(1 << 15)
    arena = DeviceArena()
    from gpu_helpers import materialize
    packed, h = materialize(inst, arena)
    with Runtime(arena, pool_size=2, policy=Fixed(5), fetch="device") as rt:
        tasks = [rt.launch(routines.get("vecadd"), Dim3(inst.grid.x), Dim3(256), 0, packed) for _ in range(7)]
        rt.device_synchronize()
        c = rt.counters
    nf = -(-inst.grid.x // 5)
    assert all(t.fetches == nf and t.remaining == 0 for t in tasks)
    assert c.fetch_count == 7 * nf and c.blocks_executed == 7 * inst.grid.x
    want, _ = oracle.run(inst)
    assert bit_equal(arena.to_numpy(h["c"]), want["c"])


@gpu
@pytest.mark.parametrize("grain", [1, 2, 7])
def test_device_fetch_jit_kernels_vs_oracle(need_gpu, reference, grain):
    """Every corpus kernel forced through the JIT (codegen.py) with device
    fetching: the generated kernel's persistent CTAs claim fetches."""
    from paper_2206_07896_b200 import routines as R
    R.FORCE_JIT = True
    try:
        rng = random.Random(77 + grain)
        for name, make in I.CORPUS.items():
            inst = make(rng)
            want, trap = oracle.run(inst)
            got, got_trap, task, counters = gpu_run(inst, pool_size=2, policy=Fixed(grain), instrument=True,
                                                    fetch="device")
            assert (trap is None) == (got_trap is None), (name, trap, got_trap)
            if trap is not None:
                assert got_trap[0] == trap[0], (name, trap, got_trap)
                continue
            for buf in inst.outputs:
                assert bit_equal(got[buf], want[buf]), (name, buf)
            total = inst.grid.x * inst.grid.y * inst.grid.z
            assert list(task.executed) == [1] * total
            assert counters.blocks_executed == total
    finally:
        R.FORCE_JIT = False


@gpu
def test_device_fetch_traps(need_gpu):
    """A launch the host sees trapping keeps host fetches (exact block); a
    kernel without a device-fetch body (hotspot) keeps host fetches too."""
    inst = _vecadd(4096)
    arena = DeviceArena()
    from gpu_helpers import materialize
    packed, h = materialize(inst, arena)
    short = arena.alloc("f32", 1000)
    bad = PackedArgs([ArgSlot("handle", h["a"]), ArgSlot("handle", short), ArgSlot("handle", h["c"]),
                      ArgSlot("i32", 4096)])
    with Runtime(arena, fetch="device", policy=Fixed(2)) as rt:
        rt.launch(routines.get("vecadd"), Dim3(16), Dim3(256), 0, bad)
        with pytest.raises(RuntimeFault) as ei:
            rt.device_synchronize()
        assert ei.value.trap.kind == "OutOfBounds" and ei.value.block_id == 1000 // 256
    hs = I.hotspot(64, 96, 16, 16, seed=5)
    want, _ = oracle.run(hs)
    got, trap, task, _ = gpu_run(hs, policy=Fixed(3), fetch="device")
    assert trap is None and bit_equal(got["dst"], want["dst"])


@gpu
def test_device_fetch_launch_range_and_hold(need_gpu):
    """launch_range with device fetching computes exactly [first, first+count)
    (executed[] indexed from first); hold_blocks keeps host-issued fetches
    (nothing runs before the synchronize) and still matches."""
    n = 1 << 14
    inst = _vecadd(n)
    want, _ = oracle.run(inst)
    arena = DeviceArena()
    from gpu_helpers import materialize
    packed, h = materialize(inst, arena)
    gx = inst.grid.x
    first, count = 5, gx - 9
    with Runtime(arena, fetch="device", policy=Fixed(2), instrument=True) as rt:
        task = rt.launch_range(routines.get("vecadd"), Dim3(gx), Dim3(256), 0, packed, first, count)
        rt.device_synchronize()
        assert list(task.executed) == [1] * count and task.fetches == -(-count // 2)
    got = arena.to_numpy(h["c"])
    lo, hi = first * 256, (first + count) * 256
    assert bit_equal(got[lo:hi], want["c"][lo:hi])
    assert not got[:lo].any() and not got[hi:].any()
    arena.fill_value(h["c"], 0.0)
    with Runtime(arena, fetch="device", hold_blocks=True, policy=Fixed(3)) as rt:
        task = rt.launch(routines.get("vecadd"), Dim3(gx), Dim3(256), 0, packed)
        assert not arena.to_numpy(h["c"]).any()  # held: nothing ran
        rt.device_synchronize()
        assert task.remaining == 0
    assert bit_equal(arena.to_numpy(h["c"]), want["c"])
