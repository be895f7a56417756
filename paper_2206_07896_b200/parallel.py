"""Multi-GPU block partitioning (one process per GPU).

The reference's only parallelism is block-level data parallelism: a grid's
independent blocks are handed out to pool workers in coarse ranges, the
average grain being ceil(totalBlocks / pool) (runtime.py:78-101,
PAPER.md:101-110).  Across GPUs the workers are the ranks: rank r owns the
r-th contiguous range of `ceil(total / world)` units (rows of the hotspot
grid, logical blocks of a 1D launch), and only kernels whose blocks exchange
data need a collective:

  * hotspot — row bands with ghost zones: each rank also holds `halo` rows
    of each neighbour band and recomputes them; after `halo` iterations the
    invalid region (which grows one row per iteration from a ghost edge) has
    just reached the owned rows, so `halo` rows per side are exchanged with
    NCCL point-to-point every `halo` iterations.
  * hist / hist_stride / wreduce / kmeans — per-rank partial counts or sums
    combined with one all-reduce (launch_sharded, COMBINE).
  * nn top-k (nn_topk_sharded) — each rank selects its k nearest records,
    one all-gather of k (index, distance) pairs, merged in (distance, index)
    order.
  * vecadd / nn / fir / reduce / backprop — disjoint outputs: no exchange is needed for
    the computation; launch_sharded assembles the full output on every rank
    with one all-gather when the caller wants it replicated.
  * bfs level step — monotone levels and flag: all-reduce MAX.
  * bfs whole traversal (bfs_levels_sharded) — ranks own vertex ranges and
    expand only their frontier; per level one all-gather of the nv-bit
    visited bitmap (8 MB at 2^26 vertices) merged by OR, after which every
    rank sees the same fresh set (same levels, same loop exit).

Everything here is backend-agnostic torch.distributed (NCCL on GPUs, gloo in
the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


def average_grain(total: int, world: int) -> int:
    """ceil(total / world): the Average fetch policy with ranks as workers."""
    if total < 1 or world < 1:
        raise ValueError("total and world must be >= 1")
    return -(-total // world)


def rank_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """[first, last) units owned by `rank` under the average grain."""
    g = average_grain(total, world)
    lo = min(total, rank * g)
    return lo, min(total, lo + g)


@dataclass
class HotspotBands:
    rows: int
    cols: int
    world: int
    rank: int
    halo: int = 0

    def __post_init__(self):
        self.own = rank_range(self.rows, self.world, self.rank)
        last = rank_range(self.rows, self.world, self.world - 1)
        if last[0] >= last[1]:
            # a rank without rows would leave its neighbours' halo sends
            # unmatched (the exchange would hang)
            raise ValueError(f"{self.rows} rows cannot give each of {self.world} ranks a band "
                             f"(ceil(rows / world) = {average_grain(self.rows, self.world)})")
        if self.world > 1:
            if self.halo < 1:
                raise ValueError("multi-rank hotspot needs halo >= 1")
            g = average_grain(self.rows, self.world)
            if g < self.halo:
                raise ValueError(f"band of {g} rows is thinner than the halo ({self.halo})")
        lo = max(0, self.own[0] - self.halo)
        hi = min(self.rows, self.own[1] + self.halo)
        self.local_rows = (lo, hi)

    @property
    def up(self) -> int | None:
        return self.rank - 1 if self.rank > 0 and self.own[0] > 0 else None

    @property
    def down(self) -> int | None:
        return self.rank + 1 if self.rank + 1 < self.world and self.own[1] < self.rows else None

    def own_slice(self) -> tuple[int, int]:
        """Owned rows in local row coordinates."""
        lo = self.local_rows[0]
        return self.own[0] - lo, self.own[1] - lo

    def exchanger(self, arena, stream=None) -> "HaloExchange":
        import torch

        def view(handle):
            return torch.as_tensor(arena.cuda_array(handle), device=torch.device("cuda", arena.device))
        return HaloExchange(self, view, stream)


class HaloExchange:
    """Refresh the ghost rows of a local grid from the neighbour ranks."""

    def __init__(self, bands: HotspotBands, view: Callable, stream=None):
        self.b = bands
        self.view = view
        self.stream = stream

    def exchange(self, handle) -> None:
        import torch
        import torch.distributed as dist

        b, cols, h = self.b, self.b.cols, self.b.halo
        t = self.view(handle)
        o0, o1 = b.own_slice()
        l0, l1 = 0, b.local_rows[1] - b.local_rows[0]
        ops = []
        if b.up is not None:
            ops.append(dist.P2POp(dist.isend, t[o0 * cols:(o0 + h) * cols], b.up))
            ops.append(dist.P2POp(dist.irecv, t[l0 * cols:o0 * cols], b.up))
        if b.down is not None:
            ops.append(dist.P2POp(dist.isend, t[(o1 - h) * cols:o1 * cols], b.down))
            ops.append(dist.P2POp(dist.irecv, t[o1 * cols:l1 * cols], b.down))
        if not ops:
            return
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _null()
        with ctx:
            for w in dist.batch_isend_irecv(ops):
                w.wait()


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ---------------------------------------------------------------------------
# sharded launches of the other kernels: each rank runs its block range
# (bf_launch_range), then the outputs are combined with one collective per
# buffer.  Specs name how each output buffer combines:
#   "sum"   — integer/float accumulators (atomics): ranks > 0 zero their copy
#             before the launch so the initial value is counted once, then an
#             all-reduce SUM (ints exact; f32 sums order-dependent, as the
#             reference's own atomics);
#   "max"   — monotone flags/levels (bfs: lvl only moves -1 -> cur+1, changed
#             0 -> 1): all-reduce MAX;
#   "owned" — disjoint writes: every rank keeps the values it changed, merged
#             by an all-gather of (changed mask, values) — generic over any
#             kernel whose blocks write disjoint elements.
# ---------------------------------------------------------------------------

COMBINE = {
    "vecadd": {"c": "owned"},
    "nn": {"d": "owned"},
    "reduce": {"out": "owned"},
    "fir": {"y": "owned"},
    "hist": {"counts": "sum"},
    "hist_stride": {"counts": "sum"},
    "wreduce": {"out": "sum"},
    "kmeans": {"member": "owned", "sums": "sum", "counts": "sum"},
    "bfs": {"lvl": "max", "changed": "max"},
    # backprop: blocks own disjoint weight rows (and partial-sum rows)
    "bpnn_layerforward": {"w": "owned", "partial": "owned"},
    "bpnn_adjust_weights": {"w": "owned", "oldw": "owned"},
}


class Combiner:
    """Prepare (before the rank's launch) and combine (after it) the output
    buffers of one sharded launch; tensors are 1-D torch views."""

    def __init__(self, spec: dict, world: int, rank: int):
        self.spec = spec
        self.world = world
        self.rank = rank
        self.before: dict = {}

    def prepare(self, tensors: dict) -> None:
        for name, op in self.spec.items():
            t = tensors[name]
            if op == "sum" and self.rank != 0:
                t.zero_()
            elif op == "owned":
                self.before[name] = t.clone()

    def finish(self, tensors: dict) -> None:
        import torch
        import torch.distributed as dist

        for name, op in self.spec.items():
            t = tensors[name]
            if op == "sum":
                dist.all_reduce(t, op=dist.ReduceOp.SUM)
            elif op == "max":
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            else:
                b = self.before.pop(name)
                changed = (t.view(torch.uint8).view(-1, t.element_size()) !=
                           b.view(torch.uint8).view(-1, t.element_size())).any(dim=1)
                masks = [torch.zeros_like(changed) for _ in range(self.world)]
                vals = [torch.empty_like(t) for _ in range(self.world)]
                dist.all_gather(masks, changed)
                dist.all_gather(vals, t)
                out = b.clone()
                for m, v in zip(masks, vals):
                    out[m] = v[m]
                t.copy_(out)


def launch_sharded(rt, arena, routine, grid, block, shmem: int, packed, outputs: dict,
                   world: int, rank: int):
    """Run this rank's share of a launch and combine the outputs.

    outputs: {param name: buffer handle} of the buffers the kernel writes.
    Returns the rank's KernelTask."""
    import torch
    name = getattr(routine, "name", "")
    spec = {p: op for p, op in COMBINE.get(name, {}).items() if p in outputs}
    if set(spec) != set(outputs):
        missing = set(outputs) - set(spec)
        raise ValueError(f"no combine rule for {name}: {sorted(missing)}")
    device = torch.device("cuda", arena.device)
    tensors = {p: torch.as_tensor(arena.cuda_array(h), device=device) for p, h in outputs.items()}
    comb = Combiner(spec, world, rank)
    torch.cuda.synchronize(device)
    comb.prepare(tensors)
    torch.cuda.synchronize(device)
    first, hi = rank_range(grid.x * grid.y * grid.z, world, rank)
    task = None
    if hi > first:
        task = rt.launch_range(routine, grid, block, shmem, packed, first, hi - first)
    rt.device_synchronize()
    comb.finish(tensors)
    torch.cuda.synchronize(device)
    return task


# ---------------------------------------------------------------------------
# sharded nn search: records split in contiguous ranges, each rank selects
# its k nearest (nn_topk on its own distances), one all-gather of k
# (index, distance) pairs per rank, merged by the same (distance, index)
# order — the g x k candidate merge of SURVEY §8e.
# ---------------------------------------------------------------------------

def topk_merge(idx_lists, dist_lists, k: int):
    """First k of the candidates in (distance, index) order, NaN distances
    last, -0.0 == 0.0 (kernels/nn_topk.kn); idx -1 entries are empty.
    Returns (idx int32[k] with -1 padding, dist float32[<= k])."""
    import numpy as np
    idx = np.concatenate([np.asarray(x, np.int64) for x in idx_lists]) if idx_lists else np.zeros(0, np.int64)
    dist = np.concatenate([np.asarray(x, np.float32) for x in dist_lists]) if dist_lists else np.zeros(0, np.float32)
    keep = idx >= 0
    idx, dist = idx[keep], dist[keep]
    order = np.lexsort((idx, dist))  # stable; NaN sorts last; -0.0 ties 0.0
    sel = order[:max(k, 0)]
    out = np.full(max(k, 0), -1, np.int32)
    out[:sel.size] = idx[sel]
    return out, dist[sel]


def nn_topk_sharded(local_select: Callable, n_local: int, offset: int, k: int, world: int, rank: int,
                    gather: Callable):
    """Global k nearest from per-rank picks.  local_select(k) -> (idx, dist)
    of this rank's records (local indices, -1 padded; e.g. an nn_topk launch
    on the rank's own distances); gather(idx int64[k], dist f32[k]) ->
    (world lists of both) in rank order.  Identical result on every rank."""
    import numpy as np
    idx, dist = local_select(k) if n_local > 0 else (np.full(k, -1, np.int32), np.zeros(k, np.float32))
    idx = np.asarray(idx, np.int64)
    gidx = np.where(idx >= 0, idx + offset, -1)
    d = np.zeros(k, np.float32)
    d[:np.asarray(dist).size] = np.asarray(dist, np.float32)[:k]
    if world > 1:
        il, dl = gather(gidx, d)
    else:
        il, dl = [gidx], [d]
    return topk_merge(il, dl, k)


def dist_topk_gather(device=None):
    """gather() for nn_topk_sharded over torch.distributed (NCCL tensors on
    `device`, or CPU tensors for gloo)."""
    import torch
    import torch.distributed as dist

    def gather(gidx, d):
        world = dist.get_world_size()
        ti = torch.as_tensor(gidx, dtype=torch.int64, device=device)
        td = torch.as_tensor(d, dtype=torch.float32, device=device)
        oi = [torch.empty_like(ti) for _ in range(world)]
        od = [torch.empty_like(td) for _ in range(world)]
        dist.all_gather(oi, ti)
        dist.all_gather(od, td)
        return [x.cpu().numpy() for x in oi], [x.cpu().numpy() for x in od]
    return gather


def gpu_topk_select(rt, arena, d_handle: int, n_local: int):
    """local_select() for nn_topk_sharded: one nn_topk launch over this
    rank's distance buffer."""
    from . import ArgSlot, Dim3, PackedArgs, routines

    def select(k):
        idx, dist = arena.alloc("i32", max(k, 1)), arena.alloc("f32", max(k, 1))
        rt.launch(routines.get("nn_topk"), Dim3(1), Dim3(1), 0,
                  PackedArgs([ArgSlot("handle", d_handle), ArgSlot("handle", idx), ArgSlot("handle", dist),
                              ArgSlot("i32", n_local), ArgSlot("i32", k)]))
        rt.device_synchronize()
        out = arena.to_numpy(idx)[:k], arena.to_numpy(dist)[:k]
        arena.free(idx)
        arena.free(dist)
        return out
    return select


# ---------------------------------------------------------------------------
# sharded BFS traversal
# ---------------------------------------------------------------------------

def bfs_levels_sharded(shard, row: int, col: int, lvl: int, nv: int, source: int, world: int, rank: int,
                       gather: Callable) -> int:
    """Whole traversal over `world` ranks (per-level frontier
    exchange).  `shard` provides begin/expand/merge/compact/finish/bitmap
    (graph.BfsShard on a GPU); `gather(bitmap)` returns the world bitmaps in
    rank order as one flat buffer (device pointer for the native shard).
    Returns max level + 1; `lvl` ends identical on every rank."""
    lo, hi = rank_range(nv, world, rank)
    shard.begin(source, lo, hi)
    while True:
        shard.expand(row, col)
        if world > 1:
            shard.merge(gather(shard), world)
        if shard.compact(lvl) == 0:
            break
    return shard.finish(lvl)


def nccl_bitmap_gather(world: int, device):
    """gather() for bfs_levels_sharded over torch.distributed (NCCL on GPUs):
    all_gather_into_tensor of the shard's bitmap; returns the device pointer
    of the gathered [world x words] buffer (kept alive by the closure)."""
    import torch
    import torch.distributed as dist
    state = {}

    def gather(shard):
        ptr, words = shard.bitmap()
        if "buf" not in state or state["buf"].numel() != world * words:
            state["buf"] = torch.empty(world * words, dtype=torch.int32, device=device)
        mine = _device_view(ptr, words, device)
        dist.all_gather_into_tensor(state["buf"], mine)
        torch.cuda.current_stream(device).synchronize()
        return state["buf"].data_ptr()
    return gather


def _device_view(ptr: int, n: int, device):
    """A torch int32 view of n device words at `ptr` (no copy)."""
    import torch

    class _CAI:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=device)


def nccl_allreduce(arena, device):
    """allreduce() for cluster.kmeans_iterate over torch.distributed: a list
    of arena handles is summed in place (zero-copy views); an int is summed
    and returned."""
    import torch
    import torch.distributed as dist

    def allreduce(x):
        if isinstance(x, int):
            t = torch.tensor([x], dtype=torch.int64, device=device)
            dist.all_reduce(t)
            return int(t.item())
        for h in x:
            dist.all_reduce(torch.as_tensor(arena.cuda_array(h), device=device))
        torch.cuda.current_stream(device).synchronize()
        return None
    return allreduce
