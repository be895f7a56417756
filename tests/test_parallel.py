"""Multi-rank partitioning on CPU (gloo, world sizes 2 and 3).

The GPU path runs the same `HotspotBands` / `HaloExchange` code with NCCL
and the sm_100a kernel as the step; here the step is the pinned CPU oracle,
so the test checks the partition + ghost-zone exchange protocol: the
row-banded run must equal the single-grid run bit for bit."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _hotspot_worker(rank, world, port, rows, cols, iters, halo, out_q):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import instances as I
        import oracle
        from paper_2206_07896_b200.parallel import HaloExchange, HotspotBands

        temp, power = I.hotspot_inputs(rows, cols, 3)
        params = I.hotspot_params(rows, cols)
        b = HotspotBands(rows, cols, world, rank, halo=halo)
        r0, r1 = b.local_rows
        lrows = r1 - r0
        bufs = [temp[r0 * cols:r1 * cols].copy(), np.zeros(lrows * cols, np.float32)]
        pw = power[r0 * cols:r1 * cols].copy()
        ex = HaloExchange(b, lambda h: torch.from_numpy(bufs[h]))
        cur = 0
        for it in range(iters):
            step = I.hotspot(lrows, cols, 16, 16)
            step.buffer("src").values = bufs[cur]
            step.buffer("power").values = pw
            out, trap = oracle.run(step)
            assert trap is None
            bufs[cur ^ 1][:] = out["dst"]
            cur ^= 1
            if (it + 1) % b.halo == 0 and it + 1 < iters:
                ex.exchange(cur)
        o0, o1 = b.own_slice()
        from paper_2206_07896_b200.parallel import average_grain
        g = average_grain(rows, world)
        mine = torch.zeros(g * cols, dtype=torch.float32)  # gloo gathers equal sizes
        mine[:(o1 - o0) * cols] = torch.from_numpy(bufs[cur][o0 * cols:o1 * cols])
        full = [torch.zeros(g * cols, dtype=torch.float32) for _ in range(world)]
        dist.all_gather(full, mine)
        if rank == 0:
            out_q.put(torch.cat(full).numpy()[:rows * cols])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows,cols,iters,halo", [(2, 40, 36, 7, 3), (3, 50, 20, 9, 4),
                                                        (2, 33, 16, 5, 5)])
def test_hotspot_bands_match_single_grid(world, rows, cols, iters, halo):
    import instances as I
    import oracle
    temp, power = I.hotspot_inputs(rows, cols, 3)
    want = oracle.hotspot_iterate(temp, power, rows, cols, I.hotspot_params(rows, cols), iters)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hotspot_worker, args=(r, world, port, rows, cols, iters, halo, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=90)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_rank_ranges_follow_average_grain():
    from paper_2206_07896_b200.parallel import average_grain, rank_range
    for total in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            g = average_grain(total, world)
            covered = []
            for r in range(world):
                lo, hi = rank_range(total, world, r)
                assert hi - lo <= g
                covered += list(range(lo, hi))
            assert covered == list(range(total))


def test_band_validation():
    from paper_2206_07896_b200.parallel import HotspotBands
    with pytest.raises(ValueError):
        HotspotBands(16, 16, 2, 0, halo=0)
    with pytest.raises(ValueError):
        HotspotBands(16, 16, 4, 0, halo=8)  # bands of 4 rows < halo
    with pytest.raises(ValueError):
        HotspotBands(9, 16, 4, 0, halo=1)  # ceil(9/4) = 3: rank 3 would own no rows
    b = HotspotBands(100, 8, 4, 1, halo=5)
    assert b.own == (25, 50) and b.local_rows == (20, 55) and b.up == 0 and b.down == 2


def _shard_worker(rank, world, port, out_q):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import random as _r

        import instances as I
        import oracle
        from paper_2206_07896_b200.parallel import COMBINE, Combiner, owned_ranges, rank_range
        rng = _r.Random(77)
        cases = [I.vecadd(rng), I.reduce(rng), I.hist(rng), I.wreduce(rng), I.nn(3000, 128, seed=4),
                 I.kmeans(1500, 8, 5, 128, seed=5), I.bfs(4000, 4, cur=0, seed=6, block=128),
                 I.backprop_forward(160, seed=7), I.backprop_adjust(96, seed=8)]
        results = []
        for inst in cases:
            first, hi = rank_range(inst.grid.total, world, rank)
            spec = COMBINE[inst.kernel]
            # this rank's buffers start from the instance's initial values
            init = {b.name: torch.from_numpy(np.array(b.values, dtype=oracle._NP[b.scalar]).reshape(-1)[: b.length].copy())
                    for b in inst.buffers}
            from paper_2206_07896_b200 import routines as _routines
            pnames = [p[0] for p in _routines.get(inst.kernel).params]
            scal = {pn: a[1] for pn, a in zip(pnames, inst.args) if a[0] != "buf"}
            ranges = {n: owned_ranges(inst.kernel, n, inst.grid, inst.block, scal, init[n].numel(), world)
                      for n, op in spec.items() if op == "owned"}
            # the contiguous owned-range combine covers every 1-D case here
            assert all(r is not None for r in ranges.values()), (inst.kernel, ranges)
            comb = Combiner(spec, world, rank, ranges)
            tens = {n: init[n] for n in spec}
            comb.prepare(tens)
            for b in inst.buffers:  # feed prepared values to the oracle run
                if b.name in tens:
                    b.values = tens[b.name].numpy()
            if hi > first:
                outs, trap = oracle.run(inst, block_range=(first, hi - first))
                assert trap is None
            else:
                outs = {b.name: init[b.name].numpy() for b in inst.buffers}
            res = {n: torch.from_numpy(np.ascontiguousarray(outs[n])) for n in spec}
            comb.before = {n: t for n, t in comb.before.items()}
            comb.finish(res)
            results.append({n: t.numpy().copy() for n, t in res.items()})
        if rank == 0:
            out_q.put(results)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_launches_match_single_launch(world):
    """Block-range shards + combine collectives == one full launch (oracle):
    owned writes (vecadd, reduce, nn, kmeans member), integer sums (hist,
    wreduce, kmeans counts), float sums within 1e-4, monotone max (bfs)."""
    import random as _r

    import instances as I
    import oracle
    rng = _r.Random(77)
    cases = [I.vecadd(rng), I.reduce(rng), I.hist(rng), I.wreduce(rng), I.nn(3000, 128, seed=4),
             I.kmeans(1500, 8, 5, 128, seed=5), I.bfs(4000, 4, cur=0, seed=6, block=128),
                 I.backprop_forward(160, seed=7), I.backprop_adjust(96, seed=8)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2206_07896_b200.parallel import COMBINE
    for inst, res in zip(cases, got):
        want, trap = oracle.run(inst)
        assert trap is None
        for name in COMBINE[inst.kernel]:
            w, g = want[name], res[name]
            if inst.kernel == "kmeans" and name == "sums":
                assert np.allclose(g, w, rtol=1e-4, atol=1e-4), inst.kernel
            else:
                assert np.array_equal(g.view(np.uint8), w.view(np.uint8)), (inst.kernel, name)


def _stride_worker(rank, world, port, out_q):
    """fir / hist_stride split by element ranges (parallel.stride_plan): the
    rank runs the unchanged kernel (oracle) on its views, then the owned-y
    gather or the counts all-reduce (Combiner)."""
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import instances as I
        import oracle
        from paper_2206_07896_b200 import routines
        from paper_2206_07896_b200.parallel import STRIDE_SPLIT, Combiner, stride_plan
        results, worked = [], []
        for inst in _stride_cases(I):
            pnames = [p[0] for p in routines.get(inst.kernel).params]
            scal = {pn: a[1] for pn, a in zip(pnames, inst.args) if a[0] != "buf"}
            arrays = {b.name: np.array(b.values, dtype=oracle._NP[b.scalar]).reshape(-1)[:b.length].copy()
                      for b in inst.buffers}
            lengths = {n: a.size for n, a in arrays.items()}
            bx = inst.block.x
            j0, j1, plan, owned = stride_plan(inst.kernel, bx, scal, lengths, world, rank)
            count_param, _, combine = STRIDE_SPLIT[inst.kernel]
            tens = {n: torch.from_numpy(arrays[n]) for n in combine}
            comb = Combiner(combine, world, rank, owned)
            comb.prepare(tens)
            worked.append(j1 - j0)
            if j1 > j0:
                sub = I.Instance(inst.kernel, inst.grid, inst.block, inst.shmem, [], [], inst.outputs)
                for b in inst.buffers:
                    if b.name in plan:
                        f, ln = plan[b.name]
                        sub.buffers.append(I.Buf(b.name, b.scalar, ln, arrays[b.name][f:f + ln].copy()))
                    else:
                        sub.buffers.append(I.Buf(b.name, b.scalar, b.length, arrays[b.name].copy()))
                sub.args = [("i32", j1 - j0) if (a[0] != "buf" and pn == count_param) else a
                            for pn, a in zip(pnames, inst.args)]
                out, trap = oracle.run(sub)
                assert trap is None
                for n in combine:
                    if n in plan:
                        f, ln = plan[n]
                        arrays[n][f:f + ln] = out[n]
                    else:
                        arrays[n][:] = out[n]
            comb.finish(tens)
            results.append({n: arrays[n].copy() for n in combine})
        out_q.put((rank, results, worked))
    finally:
        dist.destroy_process_group()


def _stride_cases(I):
    import random as _r
    rng = _r.Random(91)
    cases = [I.fir(rng) for _ in range(4)] + [I.hist_stride(rng) for _ in range(4)]
    # ragged block widths (views must stay 16 B aligned) and a long loop
    n = 37 * 41
    x = np.random.default_rng(5).uniform(-1, 1, n + 7).astype(np.float32)
    w = np.random.default_rng(6).uniform(-1, 1, 8).astype(np.float32)
    cases.append(I.Instance("fir", I.Geom(1), I.Geom(37), 0,
                            [I.Buf("x", "f32", x.size, x), I.Buf("y", "f32", n, np.zeros(n, np.float32)),
                             I.Buf("w", "f32", 8, w)],
                            [("buf", "x"), ("buf", "y"), ("buf", "w"), ("i32", 8), ("i32", 41)], ["y"]))
    pix = np.random.default_rng(7).integers(0, 1 << 16, 64 * 300).astype(np.int32)
    cases.append(I.Instance("hist_stride", I.Geom(1), I.Geom(64), 0,
                            [I.Buf("pix", "i32", pix.size, pix), I.Buf("counts", "i32", 13, np.zeros(13, np.int32))],
                            [("buf", "pix"), ("buf", "counts"), ("i32", 300), ("i32", 13)], ["counts"]))
    return cases


@pytest.mark.parametrize("world", [2, 3])
def test_stride_sharded_fir_hist_stride(world):
    """Grid-1 grid-stride kernels split by element ranges across ranks equal
    the single launch bit for bit, and ranks > 0 do part of the work."""
    import instances as I
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_stride_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (res, wk)) for r, res, wk in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cases = _stride_cases(I)
    for k, inst in enumerate(cases):
        want, trap = oracle.run(inst)
        if trap is not None:
            continue
        for r in range(world):
            for n, arr in got[r][0][k].items():
                assert np.array_equal(arr.view(np.uint8), want[n].view(np.uint8)), (k, r, inst.kernel, n)
    assert sum(got[r][1][k] for r in range(1, world) for k in range(len(cases))) > 0


# ---- sharded BFS traversal (parallel.bfs_levels_sharded) --------------------

class NumpyBfsShard:
    """CPU restatement of one bf_bfs_shard (TEST INFRASTRUCTURE): whole
    visited bitmap (uint32 words, bit i of word w = vertex 32w + i, 64 words
    of zero padding) and levels, expansion of the owned frontier only."""

    def __init__(self, nv):
        self.nv = nv
        self.words = (nv + 31) // 32

    def _bits(self):
        return np.unpackbits(self.now.view(np.uint8), bitorder="little")[:self.nv].astype(bool)

    def _set_bits(self, b):
        packed = np.packbits(b.astype(np.uint8), bitorder="little")
        self.now[:] = 0
        self.now.view(np.uint8)[:packed.size] = packed

    def begin(self, src, lo, hi):
        self.lo, self.hi = lo, hi
        self.now = np.zeros(self.words + 64, np.uint32)
        b = np.zeros(self.nv, bool)
        b[src] = True
        self._set_bits(b)
        self.prev = b.copy()
        self.lv = np.full(self.nv, -1, np.int32)
        self.lv[src] = 0
        self.q = [src] if lo <= src < hi else []
        self.depth = 0

    def expand(self, row, col):
        b = self._bits()
        for u in self.q:
            b[col[row[u]:row[u + 1]]] = True
        self._set_bits(b)

    def bitmap_tensor(self, world):
        from paper_2206_07896_b200.parallel import bitmap_slices
        return torch.from_numpy(self.now[:world * bitmap_slices(self.words, world)].view(np.int32))

    def merge_slice(self, recv, world, first, count):
        r = recv.numpy().view(np.uint32).reshape(world, count)
        self.now[first:first + count] = np.bitwise_or.reduce(r, axis=0)

    def set_bitmap(self, t):
        self.now[:t.numel()] = t.numpy().view(np.uint32)

    def compact(self, lvl):
        b = self._bits()
        fresh = b & ~self.prev
        self.prev = b.copy()
        ids = np.flatnonzero(fresh)
        self.lv[ids] = self.depth + 1
        self.q = [int(v) for v in ids if self.lo <= v < self.hi]
        self.depth += 1
        return int(ids.size)

    def finish(self, lvl):
        return self.depth


def _bfs_shard_worker(rank, world, port, out_q):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import instances as I
        from paper_2206_07896_b200.parallel import bfs_levels_sharded, bitmap_exchange
        results = []
        for nv, deg, seed, src in [(3000, 3, 1, 0), (5000, 8, 2, 4321), (400, 1, 3, 7)]:
            row, col = I.random_graph(nv, deg, seed)
            shard = NumpyBfsShard(nv)
            depth = bfs_levels_sharded(shard, row, col, None, nv, src, world, rank, bitmap_exchange(world, rank))
            results.append((shard.lv.copy(), depth))
        allres = [None] * world
        dist.all_gather_object(allres, results)
        if rank == 0:
            out_q.put(allres)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bfs_levels_sharded_protocol(world):
    """Vertex-range shards + per-level bitmap exchange (all-to-all of slices,
    OR, all-gather: parallel.bitmap_exchange): every rank ends
    with exactly the single-process levels (oracle) and the same depth."""
    import instances as I
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bfs_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    allres = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, (nv, deg, seed, src) in enumerate([(3000, 3, 1, 0), (5000, 8, 2, 4321), (400, 1, 3, 7)]):
        row, col = I.random_graph(nv, deg, seed)
        want, depth = oracle.bfs_full(row, col, nv, src)
        for r in range(world):
            lv, d = allres[r][k]
            assert np.array_equal(lv, want), (k, r)
            assert d == depth, (k, r)


def _topk_worker(rank, world, port, out_q):
    import numpy as np
    import torch.distributed as dist

    from paper_2206_07896_b200.parallel import dist_topk_gather, nn_topk_sharded, rank_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(11)
        n = 10007
        d = np.round(rng.uniform(0, 30, n), 1).astype(np.float32)  # many ties across ranks
        d[rng.integers(0, n, 20)] = np.nan
        d[rng.integers(0, n, 20)] = -0.0
        lo, hi = rank_range(n, world, rank)
        loc = d[lo:hi]

        def select(k):  # the device kernel's contract: stable order of the local records
            o = np.argsort(loc, kind="stable")[:k]
            idx = np.full(k, -1, np.int32)
            idx[:o.size] = o
            return idx, loc[o]
        res = {}
        for k in (1, 5, 37, 3000):
            idx, dd = nn_topk_sharded(select, hi - lo, lo, k, world, rank, dist_topk_gather())
            res[k] = (idx.tolist(), dd.view(np.uint32).tolist())
        out_q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_nn_topk_sharded_merge(world):
    """g x k candidate merge over gloo == the single-device selection (a
    stable sort of all distances), identical on every rank."""
    import numpy as np
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_topk_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    rng = np.random.default_rng(11)
    n = 10007
    d = np.round(rng.uniform(0, 30, n), 1).astype(np.float32)
    d[rng.integers(0, n, 20)] = np.nan
    d[rng.integers(0, n, 20)] = -0.0
    for k in (1, 5, 37, 3000):
        want = np.argsort(d, kind="stable")[:k]
        for r in range(world):
            idx, bits = got[r][k]
            assert idx == want.tolist(), (world, r, k)
            assert bits == d[want].view(np.uint32).tolist()
