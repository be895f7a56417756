"""GPU parity: every golden instance through the C ABI on a B200, compared
with the reference interpreter's own outputs (bit-exact; kmeans float sums
within the stated tolerance because float atomics are order-dependent)."""

import numpy as np
import pytest

import golden
import oracle
from conftest import has_gpu
from gpu_helpers import bit_equal, gpu_run, registered

pytestmark = pytest.mark.gpu

# kmeans: the reference accumulates f32 sums sequentially in (block, thread)
# order (atomic_add on an f32 buffer rounds at every store); the device sums
# in a different order, so sums get |x - y| <= 1e-4 * max(|x|, |y|, 1).
SUMS_RTOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")


def check_case(name, k, inst, expected, trap, got, got_trap):
    if trap is not None:
        assert got_trap is not None and got_trap[0] == trap, (name, k, trap, got_trap)
        return
    assert got_trap is None, (name, k, inst.kernel, got_trap)
    for buf, want in expected.items():
        g = got[buf]
        if inst.kernel == "kmeans" and buf == "sums":
            scale = np.maximum(np.maximum(np.abs(g), np.abs(want)), 1.0)
            assert np.all(np.abs(g.astype(np.float64) - want) <= SUMS_RTOL * scale), (name, k)
        else:
            assert bit_equal(g, want), (name, k, inst.kernel, buf,
                                        np.flatnonzero(g != want)[:10])


@pytest.mark.parametrize("name", golden.SETS)
def test_golden_sets_on_gpu(name):
    reg = registered()
    cases = [c for c in golden.load(name) if c[0].kernel in reg]
    if not cases:
        pytest.skip(f"no registered kernel in {name}")
    for k, (inst, expected, trap) in enumerate(cases):
        if not handwritten_geometry(inst):
            # the hand-written kernel refuses it loudly (no fallback)
            from paper_2206_07896_b200._lib import E_UNSUPPORTED, BfError
            with pytest.raises(BfError) as ei:
                gpu_run(inst)
            assert ei.value.code == E_UNSUPPORTED
            continue
        got, got_trap, _, _ = gpu_run(inst)
        check_case(name, k, inst, expected, trap, got, got_trap)


def handwritten_geometry(inst) -> bool:
    """Geometries the hand-written kernels implement."""
    if inst.kernel.startswith("bpnn_"):
        return ((inst.block.x, inst.block.y, inst.block.z) == (16, 16, 1) and inst.grid.x == 1
                and inst.grid.z == 1)
    return True


@pytest.mark.parametrize("n_in", [16, 65536, 65536 * 3 + 16])
def test_backprop_vs_oracle(n_in):
    """Rodinia backprop's device kernels at Rodinia's default input layer
    (65536 units) and ragged sizes: weights, partial sums and the adjusted
    weights / momentum bit-exact; then a forward -> adjust chain."""
    import instances as I
    fw = I.backprop_forward(n_in, seed=n_in % 97)
    want, trap = oracle.run(fw)
    got, got_trap, _, _ = gpu_run(fw)
    assert trap is None and got_trap is None
    for b in ("w", "partial"):
        assert bit_equal(got[b], want[b]), b
    adj = I.backprop_adjust(n_in, seed=n_in % 89)
    adj.buffer("w").values = want["w"]
    want2, trap = oracle.run(adj)
    got2, got_trap, _, _ = gpu_run(adj)
    assert trap is None and got_trap is None
    for b in ("w", "oldw"):
        assert bit_equal(got2[b], want2[b]), b


@pytest.mark.parametrize("pool,grain", [(1, None), (2, 1), (4, 3), (3, "avg")])
def test_pools_and_grains_match_oracle(pool, grain):
    """Fetch splitting over several worker streams changes nothing."""
    from paper_2206_07896_b200 import Average, Fixed
    reg = registered()
    policy = Average() if grain in (None, "avg") else Fixed(grain)
    cases = [c for c in golden.load("corpus_sweep") if c[0].kernel in reg][::7]
    for k, (inst, expected, trap) in enumerate(cases):
        got, got_trap, task, counters = gpu_run(inst, pool_size=pool, policy=policy, instrument=True)
        check_case("pools", k, inst, expected, trap, got, got_trap)
        total = inst.grid.total
        assert task.executed == [1] * total
        assert counters.blocks_executed == total
        assert sum(counters.busy_blocks) == total
        assert task.fetches == -(-total // task.block_per_fetch)


def test_random_instances_vs_oracle():
    """Fresh seeded instances (not in the goldens) against the pinned oracle."""
    import random
    import instances as I
    reg = registered()
    rng = random.Random(123)
    for name in I.CORPUS:
        if name not in reg:
            continue
        for _ in range(20):
            inst = I.CORPUS[name](rng)
            want, trap = oracle.run(inst)
            got, got_trap, _, _ = gpu_run(inst)
            check_case("random", 0, inst, {b: want[b] for b in inst.outputs}, trap[0] if trap else None,
                       got, got_trap)


def test_hotspot_sizes_vs_oracle():
    import instances as I
    if "hotspot" not in registered():
        pytest.skip()
    for rows, cols, bx, by in [(128, 256, 16, 16), (130, 260, 32, 8), (64, 64, 64, 1),
                               (255, 257, 16, 16), (1, 4, 4, 1), (512, 512, 128, 2)]:
        inst = I.hotspot(rows, cols, bx, by, seed=rows)
        want, trap = oracle.run(inst)
        got, got_trap, _, _ = gpu_run(inst)
        assert trap is None and got_trap is None
        assert bit_equal(got["dst"], want["dst"]), (rows, cols, bx, by)


def test_kmeans_vs_oracle_screen_and_ties():
    """f32 screen + exact f64 re-check: membership and counts bit-exact over
    shapes that hit the fast path (nf <= 32), the generic path (nf > 32),
    duplicated centroids (exact ties), tiny k and huge coordinates."""
    import instances as I
    cases = [I.kmeans(3000, 32, 16, 256, seed=11), I.kmeans(2000, 7, 5, 128, seed=12),
             I.kmeans(1500, 33, 4, 256, seed=13), I.kmeans(999, 16, 16, 96, seed=14, dup=True),
             I.kmeans(500, 3, 1, 64, seed=15), I.kmeans(4096, 32, 16, 256, seed=16, dup=True),
             I.kmeans(2000, 4, 13, 128, seed=18), I.kmeans(3001, 32, 7, 256, seed=19, dup=True)]
    big = I.kmeans(1024, 8, 6, 128, seed=17)
    f = big.buffer("f")
    f.values = (np.asarray(f.values) * 1e6 - 3e5).astype(np.float32)  # large, signed
    c = big.buffer("cent")
    c.values = np.ascontiguousarray(np.asarray(f.values).reshape(8, 1024)[:, :6].T).reshape(-1)
    cases.append(big)
    # tensor-core screen edge cases (nf = 32, k = 16, npts % 4 == 0): a centroid
    # one ulp away from another (near-ties), subnormal-scale points, and
    # non-finite features (the reference scan's NaN semantics)
    edge = I.kmeans(2048, 32, 16, 256, seed=20)
    c = np.asarray(edge.buffer("cent").values).copy()
    c[2 * 32:3 * 32] = c[:32]
    c[2 * 32 + 5] = np.nextafter(c[5], np.float32(2))
    c[3 * 32:4 * 32] = c[32:64]
    c[3 * 32 + 31] = np.nextafter(c[32 + 31], np.float32(-2))
    edge.buffer("cent").values = c
    fe = np.asarray(edge.buffer("f").values).copy().reshape(32, 2048)
    fe[:, 100:140] *= np.float32(1e-30)
    fe[3, 7] = np.nan
    fe[0, 9] = np.inf
    fe[:, 11] = np.float32(3e38)
    fe[:, 13] = c[:32]  # a point exactly on centroid 0 (= centroid 2 but one ulp)
    edge.buffer("f").values = fe.reshape(-1)
    cases.append(edge)
    for k, inst in enumerate(cases):
        want, trap = oracle.run(inst)
        got, got_trap, _, _ = gpu_run(inst)
        assert trap is None and got_trap is None
        assert bit_equal(got["member"], want["member"]), k
        assert bit_equal(got["counts"], want["counts"]), k
        w, g = want["sums"].astype(np.float64), got["sums"].astype(np.float64)
        fin = np.isfinite(w)
        assert np.array_equal(np.isnan(w), np.isnan(g)) and np.array_equal(w[np.isinf(w)], g[np.isinf(w)]), k
        w, g = w[fin], g[fin]
        assert np.all(np.abs(w - g) <= SUMS_RTOL * np.maximum(np.maximum(abs(w), abs(g)), 1.0)), k


def test_bfs_levels_vs_oracle():
    """Every level launch of several traversals, bit-exact (levels and flag)."""
    import instances as I
    for nv, deg, seed in [(5000, 4, 1), (20000, 8, 2), (777, 1, 3), (3000, 13, 4)]:
        lvl = None
        for cur in range(200):
            inst = I.bfs(nv, deg, cur=cur, seed=seed, block=256, lvl=lvl)
            want, _ = oracle.run(inst)
            got, got_trap, _, _ = gpu_run(inst)
            assert got_trap is None
            assert bit_equal(got["lvl"], want["lvl"]) and bit_equal(got["changed"], want["changed"])
            lvl = want["lvl"]
            if want["changed"][0] == 0:
                break


def test_nn_vs_oracle():
    import instances as I
    for n, blk, seed in [(100000, 256, 1), (12345, 100, 2), (7, 3, 3)]:
        inst = I.nn(n, blk, seed=seed, target=(12.5, -77.25))
        want, _ = oracle.run(inst)
        got, got_trap, _, _ = gpu_run(inst)
        assert got_trap is None and bit_equal(got["d"], want["d"])


def test_large_random_corpus_vs_oracle():
    """Bigger-than-golden shapes through the vectorised fast paths."""
    import instances as I
    rng = np.random.default_rng(5)
    n = 1 << 18
    pix = rng.integers(0, 1 << 16, n).astype(np.int32)
    for nbins in (16, 7, 32, 33, 1000, 9000):
        inst = I.Instance("hist", I.Geom(n // 256), I.Geom(256), 0,
                          [I.Buf("pix", "i32", n, pix), I.Buf("counts", "i32", nbins, np.zeros(nbins, np.int32))],
                          [("buf", "pix"), ("buf", "counts"), ("i32", n - 5), ("i32", nbins)], ["counts"])
        want, _ = oracle.run(inst)
        got, trap, _, _ = gpu_run(inst)
        assert trap is None and bit_equal(got["counts"], want["counts"]), nbins
    inst = I.Instance("reduce", I.Geom(n // 256), I.Geom(256), 0,
                      [I.Buf("x", "i32", n, pix), I.Buf("out", "i32", n // 256, np.zeros(n // 256, np.int32))],
                      [("buf", "x"), ("buf", "out"), ("i32", n - 3)], ["out"])
    want, _ = oracle.run(inst)
    got, trap, _, _ = gpu_run(inst)
    assert trap is None and bit_equal(got["out"], want["out"])
    for bx in (256, 96, 100):
        inst = I.Instance("wreduce", I.Geom(n // bx), I.Geom(bx), 0,
                          [I.Buf("x", "i32", n, pix), I.Buf("out", "i32", 1, np.zeros(1, np.int32))],
                          [("buf", "x"), ("buf", "out"), ("i32", n - 77)], ["out"])
        want, _ = oracle.run(inst)
        got, trap, _, _ = gpu_run(inst)
        assert trap is None and bit_equal(got["out"], want["out"]), bx
    x = rng.uniform(-1, 1, n + 16).astype(np.float32)
    for taps, bx, m in ((8, 256, 1024), (13, 64, 999), (1, 256, 7), (20, 128, 33), (9, 100, 37),
                        (10, 33, 41), (3, 7, 5), (9, 3, 1)):
        w = rng.uniform(-1, 1, taps).astype(np.float32)
        nout = bx * m
        inst = I.Instance("fir", I.Geom(1), I.Geom(bx), 0,
                          [I.Buf("x", "f32", nout + taps, x[:nout + taps]),
                           I.Buf("y", "f32", nout, np.zeros(nout, np.float32)), I.Buf("w", "f32", taps, w)],
                          [("buf", "x"), ("buf", "y"), ("buf", "w"), ("i32", taps), ("i32", m)], ["y"])
        want, _ = oracle.run(inst)
        got, trap, _, _ = gpu_run(inst)
        assert trap is None and bit_equal(got["y"], want["y"]), taps


def test_bfs_levels_fused_vs_oracle():
    """The fused traversal (bf_bfs_levels) gives exactly the levels of the
    per-level launches (oracle full traversal)."""
    import instances as I
    from gpu_helpers import materialize
    from paper_2206_07896_b200 import DeviceArena, Runtime, graph
    graphs = [(I.random_graph(nv, deg, seed), nv, src)
              for nv, deg, seed, src in [(5000, 4, 1, 0), (200000, 8, 2, 17), (777, 1, 3, 5), (3000, 13, 4, 2999)]]
    # variable degrees (unaligned adjacency starts) and a 700-vertex chain with
    # side branches: depth > 255 exercises the levels beyond the byte array
    g = np.random.default_rng(9)
    nv = 50000
    degs = g.integers(0, 13, nv)
    row = np.concatenate([[0], np.cumsum(degs)]).astype(np.int32)
    col = g.integers(0, nv, int(row[-1])).astype(np.int32)
    graphs.append(((row, col), nv, 3))
    # large enough for the bucketed levels (> 2 slices of 2^18 vertices),
    # variable degrees 0..16
    nv = 1 << 20
    degs = g.integers(0, 17, nv)
    row = np.concatenate([[0], np.cumsum(degs)]).astype(np.int32)
    col = g.integers(0, nv, int(row[-1])).astype(np.int32)
    graphs.append(((row, col), nv, 12345))
    nv = 1400
    adj = [[i + 1] if i < 699 else [] for i in range(nv)]
    for i in range(0, 700, 7):
        adj[i].append(700 + i % 700)
        adj[700 + i % 700].append(700 + (i + 350) % 700)
    row = np.concatenate([[0], np.cumsum([len(a) for a in adj])]).astype(np.int32)
    col = np.array([v for a in adj for v in a], np.int32)
    graphs.append(((row, col), nv, 0))
    for (row, col), nv, src in graphs:
        want, depth = oracle.bfs_full(row, col, nv, src)
        arena = DeviceArena()
        hr, hc, hl = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size), arena.alloc("i32", nv)
        arena.upload_numpy(hr, row)
        arena.upload_numpy(hc, col)
        with Runtime(arena) as rt:
            got_depth = graph.bfs_levels(rt, hr, hc, hl, nv, src)
            assert bit_equal(arena.to_numpy(hl), want)
            assert got_depth == depth
            # direction-optimizing (bottom-up on the large levels)
            arena.fill_value(hl, 7)
            tg = graph.transpose(rt, hr, hc, nv)
            assert graph.bfs_levels(rt, hr, hc, hl, nv, src, transposed=tg) == depth
            assert bit_equal(arena.to_numpy(hl), want)


def test_bfs_transpose_vs_numpy():
    """bf_bfs_transpose: crow is the in-degree prefix sum and each in-list
    holds exactly the sources of the edges into that vertex (order
    unspecified); edges outside every row range are not edges; a malformed
    row or an out-of-range target is BF_E_FAULT."""
    from paper_2206_07896_b200 import DeviceArena, Runtime, graph
    from paper_2206_07896_b200._lib import E_FAULT, BfError
    g = np.random.default_rng(5)
    for nv, maxdeg in [(1, 3), (1000, 9), (70001, 17)]:
        degs = g.integers(0, maxdeg, nv)
        row = np.concatenate([[0], np.cumsum(degs)]).astype(np.int32)
        col = g.integers(0, nv, int(row[-1]) + 5).astype(np.int32)  # 5 trailing non-edges
        arena = DeviceArena()
        hr, hc = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size)
        arena.upload_numpy(hr, row)
        arena.upload_numpy(hc, col)
        with Runtime(arena) as rt:
            tg = graph.transpose(rt, hr, hc, nv)
        crow, ccol = arena.to_numpy(tg.crow), arena.to_numpy(tg.ccol)
        ne = int(row[-1])
        src = np.repeat(np.arange(nv), degs)
        dst = col[:ne].astype(np.int64)
        assert np.array_equal(crow, np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=nv))]))
        want = np.lexsort((src, dst))
        got_pairs = np.stack([np.repeat(np.arange(nv), np.diff(crow)), ccol[:ne]])
        order = np.lexsort((got_pairs[1], got_pairs[0]))
        assert np.array_equal(got_pairs[:, order], np.stack([dst[want], src[want]]))
    arena = DeviceArena()
    hr, hc = arena.alloc("i32", 4), arena.alloc("i32", 4)
    arena.upload_numpy(hr, np.array([0, 1, 2, 4], np.int32))
    arena.upload_numpy(hc, np.array([1, 2, 3, 0], np.int32))  # target 3 >= nv
    with Runtime(arena) as rt:
        with pytest.raises(BfError) as ei:
            graph.transpose(rt, hr, hc, 3)
        assert ei.value.code == E_FAULT
        arena.upload_numpy(hc, np.array([1, 2, 0, 0], np.int32))
        arena.upload_numpy(hr, np.array([0, 2, 1, 4], np.int32))  # row not monotone
        with pytest.raises(BfError) as ei:
            graph.transpose(rt, hr, hc, 3)
        assert ei.value.code == E_FAULT


@pytest.mark.parametrize("tsteps", [0, 1, 2, 3, 4, 8, 12, 16])
def test_hotspot_run_fused_vs_oracle(tsteps):
    """Temporal blocking == the per-launch ping-pong loop, bit for bit."""
    import instances as I
    from paper_2206_07896_b200 import DeviceArena, Runtime, stencil
    for rows, cols, iters in [(200, 300, 7), (64, 128, 16), (131, 257, 5), (1, 9, 3), (700, 130, 20)]:
        temp, power = I.hotspot_inputs(rows, cols, rows + cols)
        params = I.hotspot_params(rows, cols)
        want = oracle.hotspot_iterate(temp, power, rows, cols, params, iters)
        arena = DeviceArena()
        a, p, b = (arena.alloc("f32", rows * cols) for _ in range(3))
        arena.upload_numpy(a, temp)
        arena.upload_numpy(p, power)
        with Runtime(arena) as rt:
            res = stencil.hotspot_run(rt, a, p, b, rows, cols, params, iters, tsteps)
            rt.device_synchronize()
        assert bit_equal(arena.to_numpy(res), want), (rows, cols, iters, tsteps)


def test_nn_sqrt_rounding_hard_cases():
    """f32(f64 sqrt) emulation: exact squares of f32 midpoints (f32 ties),
    neighbours one f64 ulp away (double-rounding cases), binade edges."""
    import struct
    rng = np.random.default_rng(3)
    lat, x = [], []
    for _ in range(4000):
        f = np.float32(rng.uniform(1e-3, 3e2))
        nxt = np.nextafter(f, np.float32(np.inf))
        m = (float(f) + float(nxt)) / 2.0           # exact f32 midpoint (25 bits)
        for k in (-2, -1, 0, 1, 2):                 # m^2 and its f64 neighbours
            v = m
            for _ in range(abs(k)):
                v = float(np.nextafter(v, np.inf if k > 0 else -np.inf))
            lat.append(0.0)
            x.append(-v)                               # d = 0 - (-v) = v exactly
    for e in range(-20, 20):                          # binade edges
        for v in (2.0 ** e, float(np.nextafter(2.0 ** e, 0)), float(np.nextafter(2.0 ** e, 9))):
            lat.append(0.0)
            x.append(-v)
    import instances as I
    n = len(lat)
    # one launch per distinct x would be slow: x is a kernel param, so use lng
    # for the varying part instead: d = sqrt((0 - 0)^2 + (lng - y)^2) with y = 0
    ll = np.zeros(2 * n, np.float32)
    vals = np.array([-xv for xv in x])
    # lng must be f32: use the f32 values themselves (exact squares) plus the
    # double perturbation through the param path in a second pass below
    ll[1::2] = vals.astype(np.float32)
    inst = I.Instance("nn", I.Geom(-(-n // 256)), I.Geom(256), 0,
                      [I.Buf("ll", "f32", 2 * n, ll), I.Buf("d", "f32", n, np.zeros(n, np.float32))],
                      [("buf", "ll"), ("buf", "d"), ("i32", n), ("f32", 0.0), ("f32", 0.0)], ["d"])
    want, _ = oracle.run(inst)
    got, trap, _, _ = gpu_run(inst)
    assert trap is None and bit_equal(got["d"], want["d"])
    # double-valued target: lat = 0, x = -(m + k ulp64): s = v^2 rounded in f64
    for v in vals[rng.choice(len(vals), 300, replace=False)]:
        inst = I.Instance("nn", I.Geom(1), I.Geom(32), 0,
                          [I.Buf("ll", "f32", 64, np.zeros(64, np.float32)),
                           I.Buf("d", "f32", 32, np.zeros(32, np.float32))],
                          [("buf", "ll"), ("buf", "d"), ("i32", 32), ("f32", -float(v)), ("f32", 0.0)], ["d"])
        want, _ = oracle.run(inst)
        got, trap, _, _ = gpu_run(inst)
        assert trap is None and bit_equal(got["d"], want["d"]), v


def test_launch_range_covers_grid():
    """Three block-range launches tiling the grid == one full launch."""
    import random
    import instances as I
    from gpu_helpers import materialize
    from paper_2206_07896_b200 import DeviceArena, Dim3, Runtime, routines
    rng = random.Random(31)
    for make in (I.vecadd, I.hist, I.reduce, I.wreduce):
        inst = make(rng)
        want, trap = oracle.run(inst)
        arena = DeviceArena()
        packed, handles = materialize(inst, arena)
        G = inst.grid.total
        cuts = sorted({0, G // 3, (2 * G) // 3, G})
        with Runtime(arena, pool_size=2, instrument=True) as rt:
            r = routines.get(inst.kernel)
            tasks = [rt.launch_range(r, Dim3(inst.grid.x), Dim3(inst.block.x), inst.shmem, packed, a, b - a)
                     for a, b in zip(cuts, cuts[1:]) if b > a]
            rt.device_synchronize()
        for t in tasks:
            assert t.executed == [1] * t.totalBlocks
        for buf in inst.outputs:
            assert bit_equal(arena.to_numpy(handles[buf]), want[buf]), inst.kernel


def test_arena_views():
    """DeviceArena.view (bf_view): an aliasing element range under a new
    handle; kernels launched on views see exactly that range; 16 B offsets
    only; a parent with live views cannot be freed."""
    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    from paper_2206_07896_b200._lib import BfError
    arena = DeviceArena()
    n = 4096
    a, b, c = (arena.alloc("f32", n) for _ in range(3))
    x = np.arange(n, dtype=np.float32)
    arena.upload_numpy(a, x)
    arena.upload_numpy(b, 2 * x)
    va, vb, vc = (arena.view(h, 1024, 512) for h in (a, b, c))
    assert arena.length(va) == 512 and arena.scalar_type(va) == "f32"
    assert bit_equal(arena.to_numpy(va), x[1024:1536])
    with Runtime(arena) as rt:
        rt.launch(routines.get("vecadd"), Dim3(2), Dim3(256), 0,
                  PackedArgs([ArgSlot("handle", va), ArgSlot("handle", vb), ArgSlot("handle", vc),
                              ArgSlot("i32", 512)]))
        rt.device_synchronize()
    got = arena.to_numpy(c)
    want = np.zeros(n, np.float32)
    want[1024:1536] = 3 * x[1024:1536]
    assert bit_equal(got, want)
    with pytest.raises(BfError):
        arena.view(a, 1, 8)  # 4 B offset: not 16 B aligned
    with pytest.raises(BfError):
        arena.view(a, n - 4, 8)  # past the end
    with pytest.raises(BfError):
        arena.free(a)  # live view
    for v in (va, vb, vc):
        arena.free(v)
    arena.free(a)


def test_launch_sharded_single_rank_nccl():
    """parallel.launch_sharded end to end on the device (world of one, NCCL)."""
    import os
    import random
    import socket
    import torch
    import torch.distributed as dist
    import instances as I
    from gpu_helpers import materialize
    from paper_2206_07896_b200 import DeviceArena, Dim3, Runtime, routines
    from paper_2206_07896_b200.parallel import COMBINE, launch_sharded
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        rng = random.Random(41)
        cases = [I.vecadd(rng), I.hist(rng), I.kmeans(1000, 8, 4, 128, seed=2), I.reduce(rng),
                 I.backprop_adjust(96, seed=3)]
        cases += [c for c in (I.fir(rng) for _ in range(6)) if oracle.run(c)[1] is None][:2]
        cases += [I.hist_stride(rng) for _ in range(2)]
        for inst in cases:
            want, _ = oracle.run(inst)
            arena = DeviceArena()
            packed, handles = materialize(inst, arena)
            outs = {n: handles[n] for n in COMBINE[inst.kernel]}
            with Runtime(arena) as rt:
                launch_sharded(rt, arena, routines.get(inst.kernel), Dim3(inst.grid.x, inst.grid.y, inst.grid.z),
                               Dim3(inst.block.x, inst.block.y, inst.block.z), 0, packed, outs, 1, 0)
            for n in outs:
                g = arena.to_numpy(handles[n])
                if n == "sums":
                    assert np.allclose(g, want[n], rtol=1e-4, atol=1e-4)
                else:
                    assert bit_equal(g, want[n]), (inst.kernel, n)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_bfs_shards_on_one_device_vs_oracle(world):
    """The native shard steps (bf_bfs_shard_*) for `world` ranks, driven in
    lockstep in one process on one device (the bitmap all-gather is a device
    concatenation): every shard ends with the oracle's levels; the per-level
    fresh counts agree across shards."""
    import torch
    import instances as I
    from paper_2206_07896_b200 import DeviceArena, Runtime, graph
    from paper_2206_07896_b200.parallel import rank_range
    for nv, deg, seed, src in [(20000, 8, 5, 0), (3001, 2, 6, 3000), (257, 1, 7, 9)]:
        row, col = I.random_graph(nv, deg, seed)
        want, depth = oracle.bfs_full(row, col, nv, src)
        arena = DeviceArena()
        hr, hc = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size)
        arena.upload_numpy(hr, row)
        arena.upload_numpy(hc, col)
        lv = [arena.alloc("i32", nv) for _ in range(world)]
        with Runtime(arena) as rt:
            shards = [graph.BfsShard(rt, nv) for _ in range(world)]
            for r, s in enumerate(shards):
                s.begin(src, *rank_range(nv, world, r))
            while True:
                for s in shards:
                    s.expand(hr, hc)
                # the bitmap exchange (parallel.bitmap_exchange) emulated on one
                # device: all-to-all of slices, per-slice OR, all-gather
                views = [s.bitmap_tensor(world) for s in shards]
                g = views[0].numel() // world
                torch.cuda.synchronize()
                for r, s in enumerate(shards):
                    recv = torch.cat([v[r * g:(r + 1) * g] for v in views])
                    s.merge_slice(recv, world, r * g, g)
                for r in range(world):
                    for q in range(world):
                        if q != r:
                            views[q][r * g:(r + 1) * g] = views[r][r * g:(r + 1) * g]
                torch.cuda.synchronize()
                fresh = [s.compact(lv[r]) for r, s in enumerate(shards)]
                assert len(set(fresh)) == 1
                if fresh[0] == 0:
                    break
            depths = [s.finish(lv[r]) for r, s in enumerate(shards)]
            for s in shards:
                s.close()
        assert depths == [depth] * world
        for h in lv:
            assert bit_equal(arena.to_numpy(h), want)


def test_bfs_levels_sharded_nccl_world1():
    """parallel.bfs_levels_sharded end to end over NCCL (world of one)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import instances as I
    from paper_2206_07896_b200 import DeviceArena, Runtime, graph
    from paper_2206_07896_b200.parallel import bitmap_exchange, bfs_levels_sharded
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        nv, deg = 100000, 8
        row, col = I.random_graph(nv, deg, 11)
        want, depth = oracle.bfs_full(row, col, nv, 5)
        arena = DeviceArena()
        hr, hc, hl = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size), arena.alloc("i32", nv)
        arena.upload_numpy(hr, row)
        arena.upload_numpy(hc, col)
        with Runtime(arena) as rt:
            shard = graph.BfsShard(rt, nv)
            got = bfs_levels_sharded(shard, hr, hc, hl, nv, 5, 1, 0, None)
            assert got == depth
            assert bit_equal(arena.to_numpy(hl), want)
            # the NCCL exchange itself (all-to-all, slice OR, in-place all-gather)
            # driven at every level: a world of one must leave the bitmap unchanged
            ex = bitmap_exchange(1, 0)
            shard.begin(5, 0, nv)
            while True:
                shard.expand(hr, hc)
                ex(shard)
                if shard.compact(hl) == 0:
                    break
            assert shard.finish(hl) == depth
            shard.close()
        assert bit_equal(arena.to_numpy(hl), want)
    finally:
        dist.destroy_process_group()


_KMEANS_VARIANT_SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {root!r} + '/oracle', {root!r} + '/tests']
import numpy as np
import instances as I
import oracle
from gpu_helpers import bit_equal, gpu_run
cases = [I.kmeans(3000, 32, 16, 256, seed=11), I.kmeans(999, 16, 16, 96, seed=14, dup=True),
         I.kmeans(4096, 32, 16, 256, seed=16, dup=True), I.kmeans(3001, 32, 7, 256, seed=19, dup=True),
         I.kmeans(20000, 32, 16, 256, seed=21), I.kmeans(1024, 16, 5, 128, seed=22)]
edge = I.kmeans(2048, 32, 16, 256, seed=20)
c = np.asarray(edge.buffer("cent").values).copy()
c[2 * 32:3 * 32] = c[:32]
c[2 * 32 + 5] = np.nextafter(c[5], np.float32(2))
c[3 * 32:4 * 32] = c[32:64]
c[3 * 32 + 31] = np.nextafter(c[32 + 31], np.float32(-2))
edge.buffer("cent").values = c
fe = np.asarray(edge.buffer("f").values).copy().reshape(32, 2048)
fe[3, 7] = np.nan
fe[0, 9] = np.inf
fe[:, 11] = np.float32(3e38)
fe[:, 13] = c[:32]
fe[:, 100:140] *= np.float32(1e-30)
edge.buffer("f").values = fe.reshape(-1)
cases.append(edge)
for nf in (8, 16, 24):
    cases.append(I.kmeans(2052, nf, 9, 128, seed=30 + nf, dup=True))
# kmeans_tg tile bookkeeping: an odd number of 128-point tiles per CTA (a lone
# last tile), a partial last tile, few clusters (padding rows), 2 tiles per CTA
cases.append(I.kmeans(128 * 148 * 3 + 36, 32, 3, 256, seed=41))
cases.append(I.kmeans(128 * 148 * 2, 32, 16, 256, seed=42, dup=True))
cases.append(I.kmeans(128 * 150 + 4, 32, 2, 256, seed=43))
for k, inst in enumerate(cases):
    want, _ = oracle.run(inst)
    got, trap, _, _ = gpu_run(inst)
    assert trap is None, k
    assert bit_equal(got["member"], want["member"]), k
    assert bit_equal(got["counts"], want["counts"]), k
    w, g = want["sums"].astype(np.float64), got["sums"].astype(np.float64)
    fin = np.isfinite(w)
    assert np.array_equal(np.isnan(w), np.isnan(g)), k
    assert np.all(np.abs(w[fin] - g[fin]) <= 1e-4 * np.maximum(np.maximum(abs(w[fin]), abs(g[fin])), 1.0)), k
print("ok", len(cases))
"""


@pytest.mark.parametrize("variant", [2, 3, 4, 5])
def test_kmeans_variants_vs_oracle(variant):
    """Every kmeans screen stays bit-exact in membership: the register-blocked
    FFMA screen (kmeans_rb, the fallback for shapes the tensor-core kernel does
    not take; BF_KMEANS_V=2/3 with two / one CTAs per SM) and kmeans_tc (4);
    run in a subprocess because the variant is read once when the library
    loads."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ, BF_KMEANS_V=str(variant))
    r = subprocess.run([sys.executable, "-c", _KMEANS_VARIANT_SCRIPT.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().startswith("ok"), r.stderr[-2000:]


def _km_assign_oracle(fv, cent, npts, nf, k):
    import instances as I
    inst = I.kmeans(npts, nf, k, 256, seed=0)
    inst.buffer("f").values = fv
    inst.buffer("cent").values = cent
    want, trap = oracle.run(inst)
    assert trap is None
    return want


@pytest.mark.parametrize("world", [1, 2, 3])
def test_kmeans_iterate_passes_exact(world):
    """Rodinia's host loop (cluster.KmeansDriver) for `world` ranks driven in
    lockstep on one device (sums/counts all-reduced by a device add): every
    pass's membership is exactly the reference assignment under the
    centroids that pass used, counts exact, sums within 1e-4; all ranks hold
    identical centroids; the loop reaches delta == 0."""
    import torch
    import instances as I
    from paper_2206_07896_b200 import DeviceArena, Runtime
    from paper_2206_07896_b200.cluster import KmeansDriver
    dev = torch.device("cuda", 0)
    npts, nf, k = 6000, 8, 5
    fv = I.kmeans_inputs(npts, nf, seed=31)
    cent0 = np.ascontiguousarray(fv.reshape(nf, npts)[:, :k].T).reshape(-1)
    arena = DeviceArena()
    hf = arena.alloc("f32", npts * nf)
    arena.upload_numpy(hf, fv)
    hm = arena.alloc("i32", npts)
    cents = [arena.alloc("f32", k * nf) for _ in range(world)]
    for h in cents:
        arena.upload_numpy(h, cent0)
    view = lambda h: torch.as_tensor(arena.cuda_array(h), device=dev)  # noqa: E731
    with Runtime(arena) as rt:
        drv = [KmeansDriver(rt, arena, hf, cents[r], hm, npts, nf, k, world, r) for r in range(world)]
        for p in range(60):
            used = arena.to_numpy(cents[0]).copy()
            for r in range(1, world):
                assert np.array_equal(arena.to_numpy(cents[r]).view(np.uint32), used.view(np.uint32))
            for d in drv:
                d.assign()
            s = sum(view(d.sums) for d in drv)
            c = sum(view(d.counts) for d in drv)
            for d in drv:
                view(d.sums).copy_(s)
                view(d.counts).copy_(c)
            torch.cuda.synchronize()
            want = _km_assign_oracle(fv, used, npts, nf, k)
            assert bit_equal(arena.to_numpy(hm), want["member"]), p
            assert bit_equal(arena.to_numpy(drv[0].counts), want["counts"]), p
            w, g = want["sums"].astype(np.float64), arena.to_numpy(drv[0].sums).astype(np.float64)
            assert np.all(np.abs(w - g) <= 1e-4 * np.maximum(np.maximum(abs(w), abs(g)), 1.0)), p
            delta = sum(d.update() for d in drv)
            if delta == 0:
                break
        assert p > 1 and delta == 0


def test_kmeans_iterate_nccl_world1():
    """cluster.kmeans_iterate end to end (world of one over NCCL helpers)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import instances as I
    from paper_2206_07896_b200 import DeviceArena, Runtime
    from paper_2206_07896_b200.cluster import kmeans_iterate
    from paper_2206_07896_b200.parallel import nccl_allreduce
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        # 16 well-separated blobs (point p in blob p % 16): the loop converges
        # in a few passes (uniform data needs hundreds, and the order of the
        # f32 centroid-sum atomics makes that count vary run to run)
        npts, nf, k = 50000, 32, 16
        g = np.random.default_rng(33)
        centers = g.uniform(0.0, 1.0, (k, nf))
        pts = centers[np.arange(npts) % k] + g.normal(0.0, 0.02, (npts, nf))
        fv = np.ascontiguousarray(pts.T.astype(np.float32)).reshape(-1)  # feature-major
        arena = DeviceArena()
        hf, hc, hm = arena.alloc("f32", npts * nf), arena.alloc("f32", k * nf), arena.alloc("i32", npts)
        arena.upload_numpy(hf, fv)
        arena.upload_numpy(hc, np.ascontiguousarray(fv.reshape(nf, npts)[:, :k].T).reshape(-1))
        with Runtime(arena) as rt:
            passes, delta = kmeans_iterate(rt, arena, hf, hc, hm, npts, nf, k, max_iter=500, world=1, rank=0,
                                           allreduce=nccl_allreduce(arena, torch.device("cuda", 0)))
        assert passes >= 2 and delta == 0
        cent = arena.to_numpy(hc).astype(np.float64).reshape(k, nf)
        mem = arena.to_numpy(hm)
        f = fv.reshape(nf, npts).T.astype(np.float64)
        for c in range(k):  # converged: every centroid is the mean of its members
            if (mem == c).any():
                assert np.allclose(cent[c], f[mem == c].mean(0), rtol=1e-4, atol=1e-5)
    finally:
        dist.destroy_process_group()


def test_benchmark_configs_full_size_vs_oracle():
    """The BASELINE configs at their full sizes, checked against the oracle
    where it finishes in seconds (OpenMP over host cores): hotspot 8192^2
    (3 chained launches through Runtime.launch, bit-exact), nn 2^24 records
    (bit-exact), BFS 2^24 vertices x 8 through the fused driver (levels
    bit-exact), kmeans 2^20 points x 32, k = 16 (membership/counts bit-exact)."""
    import os
    import instances as I
    from gpu_helpers import materialize
    from paper_2206_07896_b200 import DeviceArena, Dim3, Runtime, graph, routines
    threads = max(1, len(os.sched_getaffinity(0)))
    # hotspot: 3 ping-pong launches of the full grid
    n, iters = 8192, 3
    temp, power = I.hotspot_inputs(n, n, 0)
    params = I.hotspot_params(n, n)
    want = oracle.hotspot_iterate(temp, power, n, n, params, iters, nthreads=threads)
    inst = I.hotspot(n, n, 16, 16, seed=0)
    arena = DeviceArena()
    packed, h = materialize(inst, arena)
    from paper_2206_07896_b200 import ArgSlot, PackedArgs
    sl = list(packed.slots)
    sl2 = [ArgSlot("handle", h["dst"]), sl[1], ArgSlot("handle", h["src"])] + sl[3:]
    with Runtime(arena) as rt:
        for it in range(iters):
            rt.launch(routines.get("hotspot"), Dim3(n // 16, n // 16), Dim3(16, 16), 0,
                      packed if it % 2 == 0 else PackedArgs(sl2))
        rt.device_synchronize()
    got = arena.to_numpy(h["dst"] if iters % 2 == 1 else h["src"])
    assert bit_equal(got, want)
    # nn 2^24 records
    nn = I.nn(1 << 24, 256, seed=5)
    want, trap = oracle.run(nn, nthreads=threads)
    got, got_trap, _, _ = gpu_run(nn)
    assert trap is None and got_trap is None and bit_equal(got["d"], want["d"])
    # BFS 2^24 x 8, fused traversal
    nv = 1 << 24
    row, col = I.random_graph(nv, 8, 7)
    lv, depth = oracle.bfs_full(row, col, nv, 0)
    arena = DeviceArena()
    hr, hc, hl = arena.alloc("i32", nv + 1), arena.alloc("i32", col.size), arena.alloc("i32", nv)
    arena.upload_numpy(hr, row)
    arena.upload_numpy(hc, col)
    with Runtime(arena) as rt:
        assert graph.bfs_levels(rt, hr, hc, hl, nv, 0) == depth
    assert bit_equal(arena.to_numpy(hl), lv)
    # kmeans 2^20 x 32, k = 16 (one assignment pass)
    km = I.kmeans(1 << 20, 32, 16, 256, seed=9)
    want, trap = oracle.run(km)
    got, got_trap, _, _ = gpu_run(km)
    assert trap is None and got_trap is None
    assert bit_equal(got["member"], want["member"]) and bit_equal(got["counts"], want["counts"])


@pytest.mark.parametrize("switch", [{"BF_BFS_ALPHA16": "1000000"}, {"BF_BFS_ALPHA16": "1"},
                                    {"BF_BFS_DO": "0"}])
def test_bfs_opt_in_levels_vs_oracle(switch):
    """The direction-optimizing traversal under other switch points stays
    bit-exact: bottom-up on every armed level (BF_BFS_ALPHA16=1000000, from
    level 3 on, including the tiny ones and a chain graph past 255 levels,
    where the bottom-up step writes lvl directly), bottom-up only on huge
    frontiers (1), and top-down only (BF_BFS_DO=0).  Run in a subprocess: the
    switches are read when the library loads."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    script = f"""
import sys
sys.path[:0] = [{root!r}, {root!r} + '/oracle', {root!r} + '/tests']
import numpy as np
import instances as I
import oracle
from gpu_helpers import bit_equal
from paper_2206_07896_b200 import DeviceArena, Runtime, graph
g = np.random.default_rng(4)
nv = 1 << 20
degs = g.integers(0, 17, nv)
row = np.concatenate([[0], np.cumsum(degs)]).astype(np.int32)
col = g.integers(0, nv, int(row[-1])).astype(np.int32)
n = 1400
adj = [[i + 1] if i < 699 else [] for i in range(n)]
for i in range(0, 700, 7):
    adj[i].append(700 + i % 700)
    adj[700 + i % 700].append(700 + (i + 350) % 700)
chain = (np.concatenate([[0], np.cumsum([len(a) for a in adj])]).astype(np.int32),
         np.array([v for a in adj for v in a], np.int32))
for (r, c), src in [((row, col), 7), (I.random_graph(1 << 21, 8, 3), 0), (chain, 0)]:
    n = r.size - 1
    want, depth = oracle.bfs_full(r, c, n, src)
    arena = DeviceArena()
    hr, hc, hl = arena.alloc("i32", n + 1), arena.alloc("i32", c.size), arena.alloc("i32", n)
    arena.upload_numpy(hr, r)
    arena.upload_numpy(hc, c)
    with Runtime(arena) as rt:
        assert graph.bfs_levels(rt, hr, hc, hl, n, src, transposed=graph.transpose(rt, hr, hc, n)) == depth
    assert bit_equal(arena.to_numpy(hl), want)
print("ok")
"""
    env = dict(os.environ, **switch)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("switch", [{"BF_BFS_RELAX": "0"}, {"BF_BFS_RELAX": "2"}, {"BF_BFS_DEFER_DIV": "1"},
                                    {"BF_BFS_DEFER_DIV": "1000000000"}])
def test_bfs_level_variants_vs_oracle(switch):
    """Per-level launch variants stay bit-exact on every level (levels and the
    changed flag): the claiming relax (BF_BFS_RELAX=0), the RED relax without
    deferred writes (2), the default with every level deferred to bfs_apply
    (BF_BFS_DEFER_DIV=1) and with none deferred.  Subprocess: the switches
    are read when the library loads."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    script = f"""
import sys
sys.path[:0] = [{root!r}, {root!r} + '/oracle', {root!r} + '/tests']
import instances as I
import oracle
from gpu_helpers import bit_equal, gpu_run
for nv, deg, seed in [(5000, 4, 1), (20000, 8, 2), (777, 1, 3), (3000, 13, 4), (100003, 6, 5)]:
    lvl = None
    for cur in range(200):
        inst = I.bfs(nv, deg, cur=cur, seed=seed, block=256, lvl=lvl)
        want, _ = oracle.run(inst)
        got, trap, _, _ = gpu_run(inst)
        assert trap is None
        assert bit_equal(got["lvl"], want["lvl"]) and bit_equal(got["changed"], want["changed"]), (nv, cur)
        lvl = want["lvl"]
        if want["changed"][0] == 0:
            break
print("ok")
"""
    env = dict(os.environ, **switch)
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("world,rows,cols,iters,halo", [(2, 300, 256, 17, 4), (3, 1030, 512, 12, 8),
                                                        (4, 8192, 1024, 9, 8)])
def test_hotspot_bands_on_one_device_vs_oracle(world, rows, cols, iters, halo):
    """The multi-GPU hotspot of bench.py (HotspotBands row bands with ghost
    zones + HaloExchange every `halo` iterations) with `world` ranks driven in
    lockstep on one device: each rank's band runs the sm_100a kernel through
    Runtime.launch, the halo transfers are HaloExchange.transfers() done as
    device copies; the owned rows equal the single-grid oracle bit for bit."""
    import torch

    import instances as I
    from paper_2206_07896_b200 import ArgSlot, DeviceArena, Dim3, PackedArgs, Runtime, routines
    from paper_2206_07896_b200.parallel import HaloExchange, HotspotBands
    temp, power = I.hotspot_inputs(rows, cols, 11)
    params = I.hotspot_params(rows, cols)
    want = oracle.hotspot_iterate(temp, power, rows, cols, params, iters)
    arena = DeviceArena()
    dev = torch.device("cuda", arena.device)
    ranks = []
    with Runtime(arena) as rt:
        for r in range(world):
            b = HotspotBands(rows, cols, world, r, halo=halo)
            lo, hi = b.local_rows
            n = (hi - lo) * cols
            h = [arena.alloc("f32", n) for _ in range(3)]  # src, power, dst
            arena.upload_numpy(h[0], temp[lo * cols:hi * cols])
            arena.upload_numpy(h[1], power[lo * cols:hi * cols])

            def pk(a, c, h=h, lr=hi - lo):
                return PackedArgs([ArgSlot("handle", a), ArgSlot("handle", h[1]), ArgSlot("handle", c),
                                   ArgSlot("i32", lr), ArgSlot("i32", cols), ArgSlot("f32", params["sdc"]),
                                   ArgSlot("f32", params["rx1"]), ArgSlot("f32", params["ry1"]),
                                   ArgSlot("f32", params["rz1"]), ArgSlot("f32", params["amb"])])
            ranks.append((b, h, [pk(h[0], h[2]), pk(h[2], h[0])], HaloExchange(b, None)))
        cur = 0
        for it in range(iters):
            for b, h, packs, _ in ranks:
                lr = b.local_rows[1] - b.local_rows[0]
                rt.launch(routines.get("hotspot"), Dim3(-(-cols // 16), -(-lr // 16)), Dim3(16, 16), 0,
                          packs[cur])
            rt.device_synchronize()
            cur ^= 1
            if (it + 1) % halo == 0 and it + 1 < iters:
                views = [torch.as_tensor(arena.cuda_array(h[2] if cur == 1 else h[0]), device=dev)
                         for _, h, _, _ in ranks]
                sends = {}
                for r, (b, h, _, ex) in enumerate(ranks):
                    for peer, (s0, s1), _ in ex.transfers():
                        sends[(r, peer)] = views[r][s0:s1].clone()
                for r, (b, h, _, ex) in enumerate(ranks):
                    for peer, _, (r0, r1) in ex.transfers():
                        views[r][r0:r1] = sends[(peer, r)]
                torch.cuda.synchronize()
        got = np.empty(rows * cols, np.float32)
        for b, h, _, _ in ranks:
            o0, o1 = b.own_slice()
            out = arena.to_numpy(h[0] if cur == 0 else h[2])
            got[b.own[0] * cols:b.own[1] * cols] = out[o0 * cols:o1 * cols]
    assert bit_equal(got, want)
