"""nn top-k indices (Rodinia nn's k-nearest selection, kernels/nn_topk.kn):
the device selection against the oracle restatement (oracle.c or_nn_topk,
pinned to the reference interpreter by tests/golden/nn_topk.npz) and, at
sizes the O(k n) oracle cannot reach quickly, against a stable sort of the
same distances (the restatement equals it on every golden instance:
test_oracle_is_a_stable_sort).  Indices bit-exact; dist bit-exact (the
selected records' own f32 distances)."""

import numpy as np
import pytest

import golden
import instances as I
import oracle
from conftest import has_gpu

gpu = pytest.mark.gpu


def _stable_topk(d: np.ndarray, n: int, k: int) -> np.ndarray:
    order = np.argsort(d[:n], kind="stable")[:k] if n > 0 else np.zeros(0, np.int64)
    out = np.full(max(k, 0), -1, np.int32)
    out[:order.size] = order
    return out


def test_oracle_is_a_stable_sort():
    """CPU: the restatement of the DSL's k passes == first k of a stable
    argsort (NaN last, -0.0 == 0.0) on every golden instance without a trap."""
    for inst, expected, trap in golden.load("nn_topk"):
        if trap is not None:
            continue
        n, k = inst.args[3][1], inst.args[4][1]
        d = np.asarray(inst.buffer("d").values, np.float32)
        want = _stable_topk(d, n, k)
        assert np.array_equal(expected["idx"][:k], want)
        got, t = oracle.run(inst)
        assert t is None and np.array_equal(got["idx"], expected["idx"])


@pytest.fixture
def need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")


def _run(d: np.ndarray, k: int, n=None, pool=1, policy=None, grid=(1,), block=(1,)):
    from gpu_helpers import gpu_run
    inst = I.nn_topk(d.size if n is None else n, k, d=d, grid=grid, block=block)
    got, trap, _, _ = gpu_run(inst, pool_size=pool, policy=policy)
    return got, trap


@gpu
@pytest.mark.parametrize("k", [1, 5, 8, 9, 16, 32, 33, 70])
def test_topk_matches_stable_sort(need_gpu, k):
    rng = np.random.default_rng(k)
    for n in (1, 3, 31, 1000, 65537, 1 << 20):
        d = np.round(rng.uniform(0, 20, n), 1).astype(np.float32)  # many exact ties
        got, trap = _run(d, k)
        assert trap is None
        want = _stable_topk(d, n, k)
        assert np.array_equal(got["idx"], want), (n, k)
        sel = want[want >= 0]
        assert np.array_equal(got["dist"][:sel.size].view(np.uint32), d[sel].view(np.uint32))


@gpu
def test_topk_specials(need_gpu):
    """NaN (sorted last, ties by index), +-inf, signed zeros (equal: index
    order; dist keeps each record's own sign), negatives, k > n."""
    rng = np.random.default_rng(3)
    for n in (10, 4097, 300001):
        d = rng.uniform(-5, 5, n).astype(np.float32)
        for p, v in zip(rng.integers(0, n, 40), [np.nan, -0.0, 0.0, np.inf, -np.inf] * 8):
            d[p] = v
        for k in (4, 17, n + 3 if n < 100 else 40):
            got, trap = _run(d, k)
            want = _stable_topk(d, n, k)
            assert trap is None and np.array_equal(got["idx"], want), (n, k)
            sel = want[want >= 0]
            assert np.array_equal(got["dist"][:sel.size].view(np.uint32), d[sel].view(np.uint32))
    d = np.full(1000, np.nan, np.float32)
    got, _ = _run(d, 12)
    assert np.array_equal(got["idx"], np.arange(12))


@gpu
def test_topk_vs_oracle_and_geometry(need_gpu):
    """The oracle on random instances, multi-block / multi-thread geometries
    (only blockIdx.x == 0 selects) and partial fetches (pool 3, Fixed(1))."""
    from paper_2206_07896_b200 import Fixed
    from gpu_helpers import bit_equal, gpu_run
    for seed, (n, k) in enumerate([(5000, 5), (2000, 20), (100, 50), (0, 4)]):
        inst = I.nn_topk(n, k, seed=seed, special=True, grid=(4, 3), block=(8, 2))
        want, wt = oracle.run(inst)
        for pool, pol in ((1, None), (3, Fixed(1)), (2, Fixed(5))):
            got, gt, task, _ = gpu_run(inst, pool_size=pool, policy=pol)
            assert gt is None and wt is None
            for b in ("idx", "dist"):
                assert bit_equal(got[b], want[b]), (seed, pool, b)


@gpu
def test_topk_traps_match_oracle(need_gpu):
    """Short idx / dist / d: OutOfBounds at the first logical block with x == 0."""
    from gpu_helpers import gpu_run
    cases = [I.nn_topk(100, 6, seed=8, idx_len=4), I.nn_topk(100, 6, seed=9, dist_len=5),
             I.nn_topk(5, 8, seed=9, dist_len=5), I.nn_topk(100, 6, seed=10, grid=(2, 2))]
    t = I.nn_topk(100, 6, seed=10)
    t.args[3] = ("i32", 120)
    cases.append(t)
    for inst in cases:
        want, wt = oracle.run(inst)
        got, gt, _, _ = gpu_run(inst)
        assert (wt is None) == (gt is None), (inst.args, wt, gt)
        if wt is not None:
            assert gt[0] == wt[0] and gt[1] == wt[1]
        else:
            assert np.array_equal(got["idx"], want["idx"])


@gpu
def test_nn_search_full_sweep_size(need_gpu):
    """nn distances + top-5 at 2^26 records (the sweep's 1 GB point) through
    Runtime.launch, against a stable sort of the downloaded distances."""
    import torch

    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    n, k = 1 << 26, 5
    arena = DeviceArena()
    ll, d, idx, dist = arena.alloc("f32", 2 * n), arena.alloc("f32", n), arena.alloc("i32", k), arena.alloc("f32", k)
    t = torch.as_tensor(arena.cuda_array(ll), device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    t[0::2].uniform_(-90, 90, generator=g)
    t[1::2].uniform_(-180, 180, generator=g)
    with Runtime(arena) as rt:
        rt.launch(routines.get("nn"), Dim3(n // 256), Dim3(256), 0,
                  PackedArgs([ArgSlot("handle", ll), ArgSlot("handle", d), ArgSlot("i32", n),
                              ArgSlot("f32", 30.0), ArgSlot("f32", 90.0)]))
        rt.launch(routines.get("nn_topk"), Dim3(1), Dim3(1), 0,
                  PackedArgs([ArgSlot("handle", d), ArgSlot("handle", idx), ArgSlot("handle", dist),
                              ArgSlot("i32", n), ArgSlot("i32", k)]))
        rt.device_synchronize()
    dv = torch.as_tensor(arena.cuda_array(d), device="cuda")
    order = torch.sort(dv, stable=True).indices[:k].cpu().numpy().astype(np.int32)
    assert np.array_equal(arena.to_numpy(idx), order)
    assert np.array_equal(arena.to_numpy(dist), dv[torch.as_tensor(order, device="cuda").long()].cpu().numpy())


@gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_topk_shards_on_one_device(need_gpu, world):
    """The sharded search's protocol with the device selection per shard
    (each shard an nn_topk launch over its own record range, merged by
    parallel.topk_merge), driven for `world` ranks in one process."""
    from paper_2206_07896_b200 import DeviceArena, Runtime
    from paper_2206_07896_b200.parallel import gpu_topk_select, nn_topk_sharded, rank_range
    rng = np.random.default_rng(world)
    n = 200003
    d = np.round(rng.uniform(0, 10, n), 2).astype(np.float32)
    d[rng.integers(0, n, 50)] = np.nan
    arena = DeviceArena()
    with Runtime(arena) as rt:
        for k in (5, 40):
            picks = []
            for r in range(world):
                lo, hi = rank_range(n, world, r)
                h = arena.alloc("f32", max(hi - lo, 1))
                if hi > lo:
                    arena.upload_numpy(h, d[lo:hi])
                sel = gpu_topk_select(rt, arena, h, hi - lo)
                picks.append(nn_topk_sharded(sel, hi - lo, lo, k, 1, 0, None))
                arena.free(h)
            from paper_2206_07896_b200.parallel import topk_merge
            idx, dd = topk_merge([p[0] for p in picks], [p[1] for p in picks], k)
            want = np.argsort(d, kind="stable")[:k]
            assert np.array_equal(idx, want), (world, k)
            assert np.array_equal(dd.view(np.uint32), d[want].view(np.uint32))
