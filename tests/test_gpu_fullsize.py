"""Parity at the BASELINE.json configs' full sizes, and the runtime's partial
fetch paths for the north-star kernels, on a B200 against the oracle.

* hotspot 8192 x 8192, 100 ping-pong launches through Runtime.launch,
  bit-exact against oracle.hotspot_iterate (OpenMP over host cores: blocks
  write disjoint cells, so the threaded oracle equals the sequential one);
* kmeans 16,777,216 points x 32 features, k = 16: membership and counts
  bit-exact (oracle or_kmeans_mt), sums within SUMS_RTOL;
* BFS 2^26 vertices x 8 out-edges: the fused traversal (graph.bfs_levels)
  and Rodinia's per-level host loop through Runtime.launch, levels
  bit-exact against oracle.bfs_full;
* every north-star kernel (hotspot, nn, nn_topk, bfs, kmeans, backprop)
  through pool sizes 2 / 3, Fixed(1..3) grains and 3-way launch_range
  tilings: any split of a launch into fetches must equal the whole launch
  (runtime.py:175-201, 323-350), and the fetch-count law holds.
"""

import os

import numpy as np
import pytest

import instances as I
import oracle
from conftest import has_gpu
from gpu_helpers import bit_equal, gpu_run, materialize, registered

pytestmark = pytest.mark.gpu
SUMS_RTOL = 1e-4
THREADS = max(1, len(os.sched_getaffinity(0)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")


def _sums_close(got, want):
    g, w = got.astype(np.float64), want.astype(np.float64)
    return bool(np.all(np.abs(g - w) <= SUMS_RTOL * np.maximum(np.maximum(np.abs(g), np.abs(w)), 1.0)))


def test_hotspot_8192_100_launches_vs_oracle():
    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    n, iters = 8192, 100
    temp, power = I.hotspot_inputs(n, n, 0)
    params = I.hotspot_params(n, n)
    want = oracle.hotspot_iterate(temp, power, n, n, params, iters, nthreads=THREADS)
    arena = DeviceArena()
    src, pw, dst = arena.alloc("f32", n * n), arena.alloc("f32", n * n), arena.alloc("f32", n * n)
    arena.upload_numpy(src, temp)
    arena.upload_numpy(pw, power)

    def pk(a, b):
        return PackedArgs([ArgSlot("handle", a), ArgSlot("handle", pw), ArgSlot("handle", b),
                           ArgSlot("i32", n), ArgSlot("i32", n), ArgSlot("f32", params["sdc"]),
                           ArgSlot("f32", params["rx1"]), ArgSlot("f32", params["ry1"]),
                           ArgSlot("f32", params["rz1"]), ArgSlot("f32", params["amb"])])
    packs = [pk(src, dst), pk(dst, src)]
    with Runtime(arena) as rt:
        for it in range(iters):
            rt.launch(routines.get("hotspot"), Dim3(n // 16, n // 16), Dim3(16, 16), 0, packs[it % 2])
        rt.device_synchronize()
    got = arena.to_numpy(src if iters % 2 == 0 else dst)
    assert bit_equal(got, want), np.flatnonzero(got != want)[:10]


def test_kmeans_16M_x32_k16_vs_oracle():
    km = I.kmeans(1 << 24, 32, 16, 256, seed=0)
    want, trap = oracle.run(km, nthreads=THREADS)
    got, got_trap, _, _ = gpu_run(km)
    assert trap is None and got_trap is None
    assert bit_equal(got["member"], want["member"]), np.flatnonzero(got["member"] != want["member"])[:10]
    assert bit_equal(got["counts"], want["counts"])
    assert _sums_close(got["sums"], want["sums"])


@pytest.fixture(scope="module")
def graph_2_26():
    nv = 1 << 26
    row, col = I.random_graph(nv, 8, 0)
    lv, depth = oracle.bfs_full(row, col, nv, 0)
    return nv, row, col, lv, depth


def _bfs_arena(nv, row, col):
    from paper_2206_07896_b200 import DeviceArena
    arena = DeviceArena()
    hr, hc, hl = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size), arena.alloc("i32", nv)
    arena.upload_numpy(hr, row)
    arena.upload_numpy(hc, col)
    return arena, hr, hc, hl


def test_bfs_2_26_fused_vs_oracle(graph_2_26):
    from paper_2206_07896_b200 import Runtime, graph
    nv, row, col, lv, depth = graph_2_26
    arena, hr, hc, hl = _bfs_arena(nv, row, col)
    with Runtime(arena) as rt:
        assert graph.bfs_levels(rt, hr, hc, hl, nv, 0) == depth
    assert bit_equal(arena.to_numpy(hl), lv)


def test_bfs_2_26_direction_optimizing_vs_oracle(graph_2_26):
    from paper_2206_07896_b200 import Runtime, graph
    nv, row, col, lv, depth = graph_2_26
    arena, hr, hc, hl = _bfs_arena(nv, row, col)
    with Runtime(arena) as rt:
        tg = graph.transpose(rt, hr, hc, nv)
        for _ in range(2):  # the second traversal reuses the scratch
            arena.fill_value(hl, 3)
            assert graph.bfs_levels(rt, hr, hc, hl, nv, 0, transposed=tg) == depth
            assert bit_equal(arena.to_numpy(hl), lv)


def test_bfs_2_26_per_level_vs_oracle(graph_2_26):
    """Rodinia's host loop: one `bfs` launch per level, read `changed`."""
    from paper_2206_07896_b200 import ArgSlot, Dim3, PackedArgs, Runtime, routines
    nv, row, col, lv, depth = graph_2_26
    arena, hr, hc, hl = _bfs_arena(nv, row, col)
    chg = arena.alloc("i32", 1)
    init = np.full(nv, -1, np.int32)
    init[0] = 0
    arena.upload_numpy(hl, init)
    cur = 0
    with Runtime(arena) as rt:
        while True:
            arena.fill_value(chg, 0)
            rt.launch(routines.get("bfs"), Dim3(nv // 256), Dim3(256), 0,
                      PackedArgs([ArgSlot("handle", hr), ArgSlot("handle", hc), ArgSlot("handle", hl),
                                  ArgSlot("handle", chg), ArgSlot("i32", nv), ArgSlot("i32", cur)]))
            rt.device_synchronize()
            if int(arena.to_numpy(chg)[0]) == 0:
                break
            cur += 1
    assert cur + 1 == depth
    assert bit_equal(arena.to_numpy(hl), lv)


# ---------------------------------------------------------------------------
# partial fetches: pools, fixed grains, launch_range tilings
# ---------------------------------------------------------------------------

def _bfs_mid_level(nv=20000, seed=3):
    """A level step with a non-trivial frontier: levels <= 2 of a traversal."""
    row, col = I.random_graph(nv, 8, seed)
    lv, _ = oracle.bfs_full(row, col, nv, 0)
    lvl = np.where((lv >= 0) & (lv <= 2), lv, -1).astype(np.int32)
    return I.bfs(nv, 8, cur=2, seed=seed, lvl=lvl)


def _north_star_cases():
    cases = {  # name -> (kernel, instance maker)
        "hotspot": ("hotspot", lambda: I.hotspot(130, 260, 16, 16, seed=5)),
        "hotspot_32x8": ("hotspot", lambda: I.hotspot(200, 300, 32, 8, seed=6)),
        "nn": ("nn", lambda: I.nn(50000, 256, seed=4)),
        "bfs": ("bfs", _bfs_mid_level),
        "kmeans": ("kmeans", lambda: I.kmeans(1 << 15, 32, 16, 256, seed=5)),
        "kmeans_nf8_k5": ("kmeans", lambda: I.kmeans(20000, 8, 5, 128, seed=6)),
        "bpnn_layerforward": ("bpnn_layerforward", lambda: I.backprop_forward(4096, seed=5)),
        "bpnn_adjust_weights": ("bpnn_adjust_weights", lambda: I.backprop_adjust(4096, seed=6)),
    }
    reg = registered()
    return {name: make for name, (kernel, make) in cases.items() if kernel in reg}


CASES = _north_star_cases() if has_gpu() else {}
_CACHE = {}


def _case(name):
    if name not in _CACHE:
        inst = CASES[name]()
        want, trap = oracle.run(inst)
        assert trap is None
        _CACHE[name] = (inst, want)
    return _CACHE[name]


def _check(inst, want, got):
    for buf in inst.outputs:
        if inst.kernel == "kmeans" and buf == "sums":
            assert _sums_close(got[buf], want[buf]), buf
        else:
            assert bit_equal(got[buf], want[buf]), (inst.kernel, buf, np.flatnonzero(got[buf] != want[buf])[:8])


@pytest.mark.parametrize("pool,grain", [(2, "avg"), (3, "avg"), (1, 1), (2, 2), (3, 3), (3, 1)])
@pytest.mark.parametrize("name", sorted(CASES))
def test_north_star_pools_and_grains_vs_oracle(name, pool, grain):
    from paper_2206_07896_b200 import Average, Fixed
    inst, want = _case(name)
    policy = Average() if grain == "avg" else Fixed(grain)
    got, got_trap, task, counters = gpu_run(inst, pool_size=pool, policy=policy, instrument=True)
    assert got_trap is None
    _check(inst, want, got)
    total = inst.grid.total
    assert task.fetches == -(-total // task.block_per_fetch)
    assert task.executed == [1] * total
    assert counters.blocks_executed == total and sum(counters.busy_blocks) == total


@pytest.mark.parametrize("pool", [1, 3])
@pytest.mark.parametrize("name", sorted(CASES))
def test_north_star_launch_range_tilings_vs_oracle(name, pool):
    """Three block ranges tiling the grid (uneven, one of them a single
    block) launched separately == the whole launch."""
    from paper_2206_07896_b200 import DeviceArena, Dim3, Runtime, routines
    inst, want = _case(name)
    arena = DeviceArena()
    packed, handles = materialize(inst, arena)
    G = inst.grid.total
    cuts = sorted({0, 1, max(1, G // 3), max(1, (2 * G) // 3 + 1), G})
    with Runtime(arena, pool_size=pool, instrument=True) as rt:
        r = routines.get(inst.kernel)
        g = Dim3(inst.grid.x, inst.grid.y, inst.grid.z)
        b = Dim3(inst.block.x, inst.block.y, inst.block.z)
        tasks = [rt.launch_range(r, g, b, inst.shmem, packed, lo, hi - lo)
                 for lo, hi in zip(cuts, cuts[1:]) if hi > lo]
        rt.device_synchronize()
    for t in tasks:
        assert t.executed == [1] * t.totalBlocks
    got = {buf: arena.to_numpy(handles[buf]) for buf in inst.outputs}
    _check(inst, want, got)
