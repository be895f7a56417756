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
    expand only their frontier; per level the nv-bit visited bitmap (8 MB at
    2^26 vertices) is OR-reduced by an all-to-all of slices, a per-slice OR
    and an all-gather (~2 bitmaps received per rank), after which every rank
    sees the same fresh set (same levels, same loop exit).

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

    def transfers(self) -> list:
        """[(peer, (send lo, hi), (recv lo, hi))] in local element offsets:
        the first `halo` owned rows go up and the ghost rows above are
        received from there; the last `halo` owned rows go down and the ghost
        rows below come back."""
        b, cols, h = self.b, self.b.cols, self.b.halo
        o0, o1 = b.own_slice()
        l0, l1 = 0, b.local_rows[1] - b.local_rows[0]
        out = []
        if b.up is not None:
            out.append((b.up, (o0 * cols, (o0 + h) * cols), (l0 * cols, o0 * cols)))
        if b.down is not None:
            out.append((b.down, ((o1 - h) * cols, o1 * cols), (o1 * cols, l1 * cols)))
        return out

    def exchange(self, handle) -> None:
        import torch
        import torch.distributed as dist

        t = self.view(handle)
        ops = []
        for peer, (s0, s1), (r0, r1) in self.transfers():
            ops.append(dist.P2POp(dist.isend, t[s0:s1], peer))
            ops.append(dist.P2POp(dist.irecv, t[r0:r1], peer))
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
#   "owned" — disjoint writes.  Where the kernel's index map sends a block
#             range to a contiguous element range (owned_ranges: 1-D launches
#             of vecadd / nn / kmeans / reduce, Rodinia's 1 x n/16 backprop
#             grid), every rank contributes exactly its range and one
#             all-gather of ceil-padded ranges assembles the buffer: each
#             rank receives about one buffer's worth, not world copies.  Other
#             geometries (duplicated threads, 2-D grids) fall back to a
#             generic all-gather of (changed mask, values).
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


def _block_span(kernel: str, buf: str, grid, block, scalars: dict, b0: int, b1: int):
    """[lo, hi) bounding every element that logical blocks [b0, b1) can
    write in `buf` (before clipping), or None when the index map is not a
    contiguous function of the block id for this geometry."""
    one_d = grid.y == 1 and grid.z == 1
    if b1 <= b0:
        return (0, 0)
    if kernel in ("vecadd", "nn", "kmeans") and buf in ("c", "d", "member"):
        # id = blockIdx.x * blockDim.x + threadIdx.x  (corpus/vecadd.kn, kernels/nn.kn, kmeans.kn)
        if one_d and block.y == 1 and block.z == 1:
            return b0 * block.x, b1 * block.x
        return None
    if kernel == "reduce" and buf == "out" and one_d:
        return b0, b1  # out[blockIdx.x] (corpus/reduce.kn)
    if kernel in ("bpnn_layerforward", "bpnn_adjust_weights") and grid.x == 1 and grid.z == 1 \
            and block.z == 1 and block.x <= 16 and block.y <= 16:
        hid = scalars["hid"]
        if hid < 0:
            return None
        if buf in ("w", "oldw"):
            # index = (hid+1)*(16*by + ty + 1) + tx + 1 (kernels/backprop.kn); adjust's block 0
            # also writes the bias row w[1..16]
            lo = (hid + 1) * (16 * b0 + 1) + 1
            if b0 == 0 and kernel == "bpnn_adjust_weights":
                lo = 1
            hi = (hid + 1) * (16 * (b1 - 1) + block.y) + block.x + 1
            return lo, hi
        if buf == "partial":
            return b0 * hid, (b1 - 1) * hid + block.y  # partial[by*hid + ty]
    return None


def owned_ranges(kernel: str, buf: str, grid, block, scalars: dict, length: int, world: int):
    """Per-rank [lo, hi) element ranges of an "owned" buffer under the
    rank_range block split, clipped to the buffer; None when the map is not
    contiguous or the ranks' ranges would overlap (then the masked combine
    is used)."""
    total = grid.x * grid.y * grid.z
    out = []
    for r in range(world):
        b0, b1 = rank_range(total, world, r)
        span = _block_span(kernel, buf, grid, block, scalars, b0, b1)
        if span is None:
            return None
        lo, hi = max(0, min(span[0], length)), max(0, min(span[1], length))
        out.append((lo, max(lo, hi)))
    nonempty = sorted(x for x in out if x[1] > x[0])
    if any(a[1] > b[0] for a, b in zip(nonempty, nonempty[1:])):
        return None
    return out


def gather_ranges(t, ranges, rank: int) -> None:
    """Replicate a 1-D tensor whose ranks each hold the final values of
    their own disjoint [lo, hi): one all-gather of ceil-padded pieces, then
    every rank writes the others' pieces in place.  Received bytes per rank
    = world x the largest piece (~ the buffer), not world x the buffer."""
    import torch
    import torch.distributed as dist
    world = len(ranges)
    width = max((hi - lo for lo, hi in ranges), default=0)
    if width == 0:
        return
    lo, hi = ranges[rank]
    send = torch.zeros(width, dtype=t.dtype, device=t.device)
    send[:hi - lo] = t[lo:hi]
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send)
    for q, (a, b) in enumerate(ranges):
        if q != rank and b > a:
            t[a:b] = parts[q][:b - a]


class Combiner:
    """Prepare (before the rank's launch) and combine (after it) the output
    buffers of one sharded launch; tensors are 1-D torch views.  `ranges`
    maps owned buffers to their per-rank element ranges (owned_ranges)."""

    def __init__(self, spec: dict, world: int, rank: int, ranges: dict | None = None):
        self.spec = spec
        self.world = world
        self.rank = rank
        self.ranges = ranges or {}
        self.before: dict = {}

    def prepare(self, tensors: dict) -> None:
        for name, op in self.spec.items():
            t = tensors[name]
            if op == "sum" and self.rank != 0:
                t.zero_()
            elif op == "owned" and self.ranges.get(name) is None:
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
            elif self.ranges.get(name) is not None:
                gather_ranges(t, self.ranges[name], self.rank)
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


def _scalars(routine, packed) -> dict:
    params = getattr(routine, "params", None) or ()
    names = [p[0] if isinstance(p, tuple) else getattr(p, "name", "") for p in params]
    return {n: s.value for n, s in zip(names, packed.slots) if s.kind != "handle"}


def launch_sharded(rt, arena, routine, grid, block, shmem: int, packed, outputs: dict,
                   world: int, rank: int):
    """Run this rank's share of a launch and combine the outputs.

    outputs: {param name: buffer handle} of the buffers the kernel writes.
    Grid-1 grid-stride kernels (fir, hist_stride) are split by element
    ranges instead (launch_sharded_strides).  Returns the rank's KernelTask."""
    import torch
    name = getattr(routine, "name", "")
    if name in STRIDE_SPLIT and grid.x * grid.y * grid.z == 1:
        return launch_sharded_strides(rt, arena, routine, block, packed, outputs, world, rank)
    spec = {p: op for p, op in COMBINE.get(name, {}).items() if p in outputs}
    if set(spec) != set(outputs):
        missing = set(outputs) - set(spec)
        raise ValueError(f"no combine rule for {name}: {sorted(missing)}")
    device = torch.device("cuda", arena.device)
    tensors = {p: torch.as_tensor(arena.cuda_array(h), device=device) for p, h in outputs.items()}
    sc = _scalars(routine, packed)
    ranges = {p: owned_ranges(name, p, grid, block, sc, arena.length(outputs[p]), world)
              for p, op in spec.items() if op == "owned"}
    comb = Combiner(spec, world, rank, ranges)
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
# grid-1 grid-stride kernels (corpus fir.kn, hist_stride.kn): the single
# logical block's loop `for j < m: ... t + j*blockDim.x ...` is split into
# contiguous j ranges (output ranges with the (taps-1) read-only
# halo for fir, element ranges + all-reduce for hist_stride).  Each rank
# runs the unchanged kernel on element-range views of the buffers
# (DeviceArena.view -> bf_view): fir reads x[j0*B, j1*B + taps - 1) and
# writes y[j0*B, j1*B); hist_stride reads pix[j0*B, j1*B) and counts into its
# own partial histogram, all-reduced.
# ---------------------------------------------------------------------------

# kernel -> (strided count param, {read/write buffer: halo elements}, combine)
STRIDE_SPLIT = {
    "fir": ("m", {"x": "taps-1", "y": 0}, {"y": "owned"}),
    "hist_stride": ("k", {"pix": 0}, {"counts": "sum"}),
}


def stride_plan(kernel: str, bx: int, scalars: dict, lengths: dict, world: int, rank: int):
    """This rank's j range and the element-range views it needs:
    -> (j0, j1, {buffer: (first, length)}, {owned buffer: per-rank ranges}).
    j ranges are whole multiples of `step` strides so that every view starts
    16 B aligned (4-byte elements: j0 * bx % 4 == 0)."""
    import math
    count_param, views, combine = STRIDE_SPLIT[kernel]
    m = max(0, scalars[count_param])
    step = 4 // math.gcd(bx, 4)
    units = -(-m // step)

    def jr(r):
        if units == 0:
            return 0, 0
        a, b = rank_range(units, world, r)
        return min(a * step, m), min(b * step, m)
    j0, j1 = jr(rank)
    plan = {}
    for buf, halo in views.items():
        h = max(0, scalars["taps"] - 1) if halo == "taps-1" else 0
        first = min(j0 * bx, lengths[buf])
        plan[buf] = (first, max(0, min(j1 * bx + h, lengths[buf]) - first))
    owned = {}
    for buf, op in combine.items():
        if op == "owned":
            owned[buf] = [(min(a * bx, lengths[buf]), min(b * bx, lengths[buf]))
                          for a, b in (jr(r) for r in range(world))]
    return j0, j1, plan, owned


def launch_sharded_strides(rt, arena, routine, block, packed, outputs: dict, world: int, rank: int):
    """Element-range shard of a grid-1 grid-stride launch (fir, hist_stride)."""
    import torch

    from . import ArgSlot, Dim3, PackedArgs
    name = routine.name
    params = [p[0] for p in routine.params]
    count_param, views, combine = STRIDE_SPLIT[name]
    if set(outputs) != set(combine):
        raise ValueError(f"{name}: outputs must be {sorted(combine)}")
    handles = {n: s.value for n, s in zip(params, packed.slots) if s.kind == "handle"}
    sc = _scalars(routine, packed)
    lengths = {n: arena.length(h) for n, h in handles.items()}
    j0, j1, plan, owned = stride_plan(name, block.x, sc, lengths, world, rank)
    device = torch.device("cuda", arena.device)
    tensors = {p: torch.as_tensor(arena.cuda_array(h), device=device) for p, h in outputs.items()}
    comb = Combiner(combine, world, rank, owned)
    torch.cuda.synchronize(device)
    comb.prepare(tensors)
    torch.cuda.synchronize(device)
    task = None
    made = []
    try:
        if j1 > j0:
            slots = []
            for pname, s in zip(params, packed.slots):
                if pname in plan:
                    v = arena.view(handles[pname], *plan[pname])
                    made.append(v)
                    slots.append(ArgSlot("handle", v))
                elif pname == count_param:
                    slots.append(ArgSlot(s.kind, j1 - j0))
                else:
                    slots.append(s)
            task = rt.launch(routine, Dim3(1), block, 0, PackedArgs(slots))
        rt.device_synchronize()
    finally:
        for v in made:
            arena.free(v)
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
                       exchange: Callable) -> int:
    """Whole traversal over `world` ranks (per-level frontier
    exchange).  `shard` provides begin/expand/compact/finish (graph.BfsShard
    on a GPU); `exchange(shard)` leaves the shard's visited bitmap equal to
    the OR of all ranks' bitmaps (bitmap_exchange: all-to-all of
    bitmap slices, OR per owned slice, all-gather).  Returns max level + 1;
    `lvl` ends identical on every rank."""
    lo, hi = rank_range(nv, world, rank)
    shard.begin(source, lo, hi)
    while True:
        shard.expand(row, col)
        if world > 1:
            exchange(shard)
        if shard.compact(lvl) == 0:
            break
    return shard.finish(lvl)


def bitmap_slices(words: int, world: int) -> int:
    """Words per rank slice of the exchange: ceil(words / world) (the
    bitmap is padded to world x slice words)."""
    return -(-words // world)


def bitmap_exchange(world: int, rank: int, stream=None):
    """exchange() for bfs_levels_sharded over torch.distributed (NCCL on
    GPUs; gloo with the CPU test shard).  The shard exposes its visited
    bitmap as world x g words, g = ceil(words / world) (bitmap_tensor), and
    rank r owns words [r*g, (r+1)*g):
      1. all_to_all_single: rank r receives every rank's copy of its slice;
      2. shard.merge_slice ORs them into its own slice (on the device:
         bf_bfs_shard_merge_slice);
      3. all-gather of the slices (in place on NCCL): every rank gets all.
    Bytes received per rank and level: 2 x (world-1)/world x the bitmap
    (8 MB at 2^26 vertices), where an all-gather of whole bitmaps would
    move (world-1) x the bitmap."""
    import torch
    import torch.distributed as dist

    def exchange(shard):
        now = shard.bitmap_tensor(world)
        g = now.numel() // world
        recv = torch.empty_like(now)
        ctx = torch.cuda.stream(stream) if (stream is not None and now.is_cuda) else _null()
        with ctx:
            dist.all_to_all_single(recv, now)
            if now.is_cuda:
                torch.cuda.current_stream(now.device).synchronize()
        shard.merge_slice(recv, world, rank * g, g)
        with ctx:
            mine = now[rank * g:(rank + 1) * g]
            if now.is_cuda:
                dist.all_gather_into_tensor(now, mine)
                torch.cuda.current_stream(now.device).synchronize()
            else:
                parts = [torch.empty_like(mine) for _ in range(world)]
                dist.all_gather(parts, mine.clone())
                shard.set_bitmap(torch.cat(parts))
    return exchange


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
