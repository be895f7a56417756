"""Generate golden vectors by running the REFERENCE interpreter itself.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_golden.py

Imports `blockfuse` read-only from /root/reference (this container only; the
reference does not exist on the GPU box) and writes
  * tests/golden/<set>.npz — inputs, geometry and reference outputs of every
    golden instance, produced by blockfuse.executor.run_reference (the
    lockstep oracle, executor.py:422-489) — and for the corpus sweep also the
    reference's thread-pool runtime result (bench.runtime_outputs) for
    comparison;
  * paper_2206_07896_b200/fingerprints.json — fingerprints of the reference's
    transform() of every implemented kernel (routines.fingerprint_of).
"""

from __future__ import annotations

import json
import random
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import instances as I  # noqa: E402

from blockfuse.arena import DeviceArena  # noqa: E402
from blockfuse.bench import CORPUS as REF_CORPUS  # noqa: E402
from blockfuse.executor import ArgSlot, run_reference  # noqa: E402
from blockfuse.hostprog import PackedArgs  # noqa: E402
from blockfuse.parser import parse_unit  # noqa: E402
from blockfuse.syntax import Dim3  # noqa: E402
from blockfuse.transform import transform  # noqa: E402

from paper_2206_07896_b200 import routines  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"

_NP = {"i32": np.int32, "i64": np.int64, "f32": np.float32, "f64": np.float64}


def ref_kernels() -> dict:
    ks = {n: REF_CORPUS[n].kernel() for n in REF_CORPUS}
    for f in sorted((ROOT / "paper_2206_07896_b200" / "kernels").glob("*.kn")):
        ks.update(parse_unit(f.read_text()))
    return ks


KERNELS = ref_kernels()


def run_ref(inst: I.Instance):
    """run_reference on a fresh reference arena; returns (outputs, trap)."""
    arena = DeviceArena()
    handles = {}
    for b in inst.buffers:
        h = arena.alloc(b.scalar, b.length)
        vals = b.values.tolist() if isinstance(b.values, np.ndarray) else b.values
        arena.fill(h, vals)
        handles[b.name] = h
    slots = [ArgSlot("handle", handles[a[1]]) if a[0] == "buf" else ArgSlot(a[0], a[1]) for a in inst.args]
    trap = None
    try:
        run_reference(KERNELS[inst.kernel], Dim3(inst.grid.x, inst.grid.y, inst.grid.z),
                      Dim3(inst.block.x, inst.block.y, inst.block.z), PackedArgs(slots), arena,
                      warp_mode=inst.kernel in I.WARP_MODE, warp_size=inst.warp_size,
                      dyn_bytes=inst.shmem)
    except Exception as e:  # Trap
        trap = (getattr(e, "kind", type(e).__name__),)
    outs = {b.name: np.array(arena.to_list(handles[b.name]), dtype=_NP[b.scalar]) for b in inst.buffers}
    return outs, trap


def pack(insts: list, path: Path, with_inputs: bool = True) -> None:
    """One npz per set: i<k>_meta (json), i<k>_in_<buf>, i<k>_out_<buf>."""
    data = {}
    t0 = time.time()
    for k, inst in enumerate(insts):
        outs, trap = run_ref(inst)
        meta = dict(kernel=inst.kernel, grid=[inst.grid.x, inst.grid.y, inst.grid.z],
                    block=[inst.block.x, inst.block.y, inst.block.z], shmem=inst.shmem,
                    warp_size=inst.warp_size,
                    buffers=[[b.name, b.scalar, b.length] for b in inst.buffers],
                    args=[list(a) for a in inst.args], outputs=inst.outputs,
                    trap=trap[0] if trap else None)
        data[f"i{k}_meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
        for b in inst.buffers:
            if with_inputs:
                data[f"i{k}_in_{b.name}"] = np.array(b.values, dtype=_NP[b.scalar])
            if with_inputs or b.name in inst.outputs:
                data[f"i{k}_out_{b.name}"] = outs[b.name]
    GOLDEN.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(path, **data)
    print(f"{path.name}: {len(insts)} instances in {time.time() - t0:.1f}s, "
          f"{path.stat().st_size / 1024:.0f} KiB")


def corpus_sets() -> None:
    # the acceptance sweep (test_acceptance.py:96-115): inputs are replayed
    # by instances.equivalence_sweep(), so only outputs are stored
    pack(I.equivalence_sweep(20260823, 50), GOLDEN / "corpus_sweep.npz", with_inputs=False)
    # hist_stride (the 7th corpus kernel) and test_bench's seed-42 instances
    rng = random.Random(42)
    extra = [I.hist_stride(rng) for _ in range(30)]
    rng = random.Random(13)  # test_acceptance.py:295-322 warp mode, block 64 / grid 4
    for _ in range(10):
        inst = I.wreduce(rng)
        inst.block = I.Geom(64)
        inst.grid = I.Geom(4)
        extra.append(inst)
    pack(extra, GOLDEN / "corpus_extra.npz", with_inputs=False)


def geometry_set() -> list:
    """Multi-dimensional grids/blocks and warp sizes (generic kernel paths)."""
    rng = random.Random(7)
    out = []
    for _ in range(4):
        inst = I.vecadd(rng)
        inst.grid, inst.block = I.Geom(max(1, inst.grid.x // 2), 2, 1), I.Geom(inst.block.x, 2, 1)
        out.append(inst)
    for _ in range(4):
        inst = I.hist(rng)
        inst.grid, inst.block = I.Geom(inst.grid.x, 1, 2), I.Geom(inst.block.x, 1, 2)
        out.append(inst)
    for _ in range(3):
        inst = I.reduce(rng)
        inst.block = I.Geom(min(inst.block.x, 128), 2, 1)
        out.append(inst)
    for ws in (4, 8, 16):
        inst = I.wreduce(rng)
        inst.warp_size = ws
        out.append(inst)
    for _ in range(3):
        inst = I.fir(rng)
        inst.grid = I.Geom(2, 1, 1)
        inst.block = I.Geom(inst.block.x, 1, 2)
        out.append(inst)
    for _ in range(2):
        inst = I.hist_stride(rng)
        inst.grid = I.Geom(3)
        out.append(inst)
    inst = I.reverse(rng)
    inst.block = I.Geom(inst.block.x, 2, 1)
    out.append(inst)
    return out


def trap_set() -> list:
    rng = random.Random(11)
    out = []
    inst = I.vecadd(rng)  # n beyond the buffers
    inst.args[3] = ("i32", inst.grid.x * inst.block.x + 10)
    for b in inst.buffers:
        b.length = max(1, b.length // 2)
        b.values = b.values[: b.length]
    out.append(inst)
    inst = I.hist(rng)  # nbins = 0 -> DivByZero
    inst.args[3] = ("i32", 0)
    inst.args[2] = ("i32", max(1, inst.args[2][1]))
    out.append(inst)
    inst = I.hist(rng)  # negative pixel -> negative bin -> OutOfBounds
    inst.buffers[0].values[0] = -5
    inst.args[2] = ("i32", max(1, inst.args[2][1]))
    out.append(inst)
    inst = I.reduce(rng)  # block > 256 overflows the shared buffer
    inst.block = I.Geom(300)
    out.append(inst)
    inst = I.reverse(rng)  # too little dynamic shared memory
    inst.shmem = 4 * (inst.block.x // 2)
    out.append(inst)
    return out


def northstar_sets() -> None:
    hs = [I.hotspot(48, 64, 16, 16, seed=1), I.hotspot(37, 50, 8, 4, seed=2),
          I.hotspot(20, 36, 32, 8, seed=3, gz=2), I.hotspot(33, 31, 7, 5, seed=4)]
    # three chained iterations (ping-pong): the reference output of launch k
    # feeds launch k+1
    chain = I.hotspot(40, 44, 16, 16, seed=5)
    cur = np.array(chain.buffer("src").values)
    for _ in range(3):
        step = I.hotspot(40, 44, 16, 16, seed=5)
        step.buffer("src").values = cur.copy()
        outs, _ = run_ref(step)
        hs.append(step)
        cur = outs["dst"]
    pack(hs, GOLDEN / "hotspot.npz")
    nn = [I.nn(1000, 128, seed=1), I.nn(777, 64, seed=2, target=(-12.25, 170.5)), I.nn(0, 32, seed=3)]
    pack(nn, GOLDEN / "nn.npz")
    pack(topk_set(), GOLDEN / "nn_topk.npz")
    km = [I.kmeans(700, 8, 5, 128, seed=1), I.kmeans(300, 32, 16, 64, seed=2),
          I.kmeans(257, 4, 3, 32, seed=3, dup=True)]
    pack(km, GOLDEN / "kmeans.npz")
    # BFS: every level launch of a full traversal (reference output of level
    # k is the input of level k+1)
    bf = []
    nv, deg = 600, 3
    lvl = None
    for cur in range(64):
        inst = I.bfs(nv, deg, cur=cur, seed=1, block=128, lvl=lvl)
        outs, _ = run_ref(inst)
        bf.append(inst)
        lvl = outs["lvl"]
        if outs["changed"][0] == 0:
            break
    pack(bf, GOLDEN / "bfs.npz")


def topk_set() -> list:
    """nn_topk (Rodinia nn's k-nearest selection): ties, NaN/inf/signed
    zeros, k beyond n, n = 0, distances from an nn launch, multi-block and
    multi-thread geometries (only blockIdx.x == 0 / threadIdx.x == 0 act),
    and out-of-range traps."""
    out = [I.nn_topk(500, 5, seed=1), I.nn_topk(400, 16, seed=2, special=True),
           I.nn_topk(40, 32, seed=3, special=True), I.nn_topk(7, 12, seed=4),
           I.nn_topk(0, 3, seed=5), I.nn_topk(300, 1, seed=6, special=True),
           I.nn_topk(200, 8, seed=7, grid=(3, 2), block=(4, 2))]
    nn = I.nn(1000, 128, seed=1)
    outs, _ = run_ref(nn)
    out.append(I.nn_topk(1000, 10, d=outs["d"]))
    out.append(I.nn_topk(100, 6, seed=8, idx_len=4))     # idx too short: OutOfBounds
    out.append(I.nn_topk(100, 6, seed=9, dist_len=5))    # dist too short: OutOfBounds
    t = I.nn_topk(100, 6, seed=10)                       # n beyond d: OutOfBounds
    t.args[3] = ("i32", 120)
    out.append(t)
    return out


def backprop_set() -> list:
    """Rodinia backprop device kernels: forward passes (with the weights
    overwritten by the tile sums), a forward -> adjust chain, geometry
    variants the lockstep semantics define (duplicated z threads), traps."""
    bp = [I.backprop_forward(64, seed=1), I.backprop_forward(160, seed=2),
          I.backprop_forward(32, seed=3, block=(16, 16, 2))]
    bp.append(I.backprop_adjust(64, seed=4))
    bp.append(I.backprop_adjust(256, seed=5))
    # chain: adjust after a forward pass on the same weights
    fw = I.backprop_forward(96, seed=6)
    outs, _ = run_ref(fw)
    adj = I.backprop_adjust(96, seed=7)
    adj.buffer("w").values = outs["w"].copy()
    bp += [fw, adj]
    # traps: input layer one unit short (last block's input read), partial too short
    t1 = I.backprop_forward(48, seed=8)
    t1.buffer("input").values = np.asarray(t1.buffer("input").values)[:48]
    t1.buffer("input").length = 48
    t2 = I.backprop_forward(48, seed=9)
    t2.buffer("partial").length = 40
    t2.buffer("partial").values = np.zeros(40, np.float32)
    t3 = I.backprop_adjust(32, seed=10)
    t3.buffer("delta").length = 16
    t3.buffer("delta").values = np.asarray(t3.buffer("delta").values)[:16]
    return bp + [t1, t2, t3]


def fingerprints() -> None:
    fps = {}
    for name in routines.names():
        mk = transform(KERNELS[name], warp_mode=name in I.WARP_MODE)
        fps[name] = routines.fingerprint_of(mk.to_dict())
    p = ROOT / "paper_2206_07896_b200" / "fingerprints.json"
    p.write_text(json.dumps(fps, indent=1, sort_keys=True) + "\n")
    print(f"{p.name}: {len(fps)} kernels")


if __name__ == "__main__":
    which = set(sys.argv[1:]) or {"fp", "corpus", "geometry", "traps", "northstar"}
    if "fp" in which:
        fingerprints()
    if "corpus" in which:
        corpus_sets()
    if "geometry" in which:
        pack(geometry_set(), GOLDEN / "geometry.npz")
    if "traps" in which:
        pack(trap_set(), GOLDEN / "traps.npz")
    if "northstar" in which:
        northstar_sets()
    if "topk" in which:
        pack(topk_set(), GOLDEN / "nn_topk.npz")
    if "backprop" in which or "northstar" in which:
        pack(backprop_set(), GOLDEN / "backprop.npz")
