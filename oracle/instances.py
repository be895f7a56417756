"""Seeded problem instances for parity tests (TEST INFRASTRUCTURE ONLY).

The corpus generators replay the reference's own random-instance generators
call for call (/root/reference/pkg/src/blockfuse/bench.py:78-180: the same
`random.Random` draws in the same order), so an instance built here from a
seed is identical to the one the reference builds from that seed —
tests/test_instances.py checks this against the reference when it is
available.  The north-star generators (hotspot, nn, kmeans, bfs) are this
repository's own; their golden outputs come from running our .kn kernels
through the reference interpreter (oracle/gen_golden.py).
"""

from __future__ import annotations

import random
import struct
from dataclasses import dataclass, field
from typing import Callable

import numpy as np


@dataclass
class Geom:
    x: int = 1
    y: int = 1
    z: int = 1

    @property
    def total(self) -> int:
        return self.x * self.y * self.z


@dataclass
class Buf:
    name: str
    scalar: str
    length: int
    values: list


@dataclass
class Instance:
    kernel: str
    grid: Geom
    block: Geom
    shmem: int
    buffers: list
    args: list  # ("buf", name) | (scalar, value)
    outputs: list
    warp_size: int = 32
    meta: dict = field(default_factory=dict)

    def buffer(self, name: str) -> Buf:
        for b in self.buffers:
            if b.name == name:
                return b
        raise KeyError(name)


# ---------------------------------------------------------------------------
# corpus generators (bench.py:78-180, replayed draw for draw)
# ---------------------------------------------------------------------------

def _rand_f32(rng: random.Random, n: int) -> list:
    return [rng.uniform(-1.0, 1.0) for _ in range(n)]


def _rand_i32(rng: random.Random, n: int) -> list:
    return [rng.randrange(0, 1 << 16) for _ in range(n)]


def vecadd(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    gx = rng.randint(1, max(1, 4096 // bx))
    n = rng.randint(0, gx * bx)
    length = max(n, 1)
    a = _rand_f32(rng, length)
    b = _rand_f32(rng, length)
    return Instance("vecadd", Geom(gx), Geom(bx), 0,
                    [Buf("a", "f32", length, a), Buf("b", "f32", length, b),
                     Buf("c", "f32", length, [0.0] * length)],
                    [("buf", "a"), ("buf", "b"), ("buf", "c"), ("i32", n)], ["c"])


def reverse(rng: random.Random) -> Instance:
    n = rng.randint(1, 512)
    return Instance("reverse", Geom(1), Geom(n), 4 * n, [Buf("d", "i32", n, _rand_i32(rng, n))],
                    [("buf", "d"), ("i32", n)], ["d"])


def reduce(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    gx = rng.randint(1, min(16, max(1, 4096 // bx)))
    n = rng.randint(0, gx * bx)
    length = max(n, 1)
    return Instance("reduce", Geom(gx), Geom(bx), 0,
                    [Buf("x", "i32", length, _rand_i32(rng, length)), Buf("out", "i32", gx, [0] * gx)],
                    [("buf", "x"), ("buf", "out"), ("i32", n)], ["out"])


def hist(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    gx = rng.randint(1, max(1, 4096 // bx))
    n = rng.randint(0, gx * bx)
    nbins = rng.randint(1, 32)
    length = max(n, 1)
    return Instance("hist", Geom(gx), Geom(bx), 0,
                    [Buf("pix", "i32", length, _rand_i32(rng, length)),
                     Buf("counts", "i32", nbins, [0] * nbins)],
                    [("buf", "pix"), ("buf", "counts"), ("i32", n), ("i32", nbins)], ["counts"])


def fir(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    m = rng.randint(1, 16)
    taps = rng.randint(1, 8)
    out_len = bx * m
    x = _rand_f32(rng, out_len + taps)
    w = _rand_f32(rng, taps)
    return Instance("fir", Geom(1), Geom(bx), 0,
                    [Buf("x", "f32", out_len + taps, x), Buf("y", "f32", out_len, [0.0] * out_len),
                     Buf("w", "f32", taps, w)],
                    [("buf", "x"), ("buf", "y"), ("buf", "w"), ("i32", taps), ("i32", m)], ["y"])


def hist_stride(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    k = rng.randint(1, 16)
    nbins = rng.randint(1, 32)
    length = bx * k
    return Instance("hist_stride", Geom(1), Geom(bx), 0,
                    [Buf("pix", "i32", length, _rand_i32(rng, length)),
                     Buf("counts", "i32", nbins, [0] * nbins)],
                    [("buf", "pix"), ("buf", "counts"), ("i32", k), ("i32", nbins)], ["counts"])


def wreduce(rng: random.Random) -> Instance:
    bx = rng.randint(1, 256)
    gx = rng.randint(1, max(1, 4096 // bx))
    n = rng.randint(0, gx * bx)
    length = max(n, 1)
    return Instance("wreduce", Geom(gx), Geom(bx), 0,
                    [Buf("x", "i32", length, _rand_i32(rng, length)), Buf("out", "i32", 1, [0])],
                    [("buf", "x"), ("buf", "out"), ("i32", n)], ["out"])


CORPUS: dict[str, Callable[[random.Random], Instance]] = {
    "vecadd": vecadd, "reverse": reverse, "reduce": reduce, "hist": hist, "fir": fir,
    "hist_stride": hist_stride, "wreduce": wreduce,
}
# the reference's equivalence suite order (bench.py:211-212)
EQUIVALENCE_CASES = ["vecadd", "reverse", "reduce", "hist", "fir", "wreduce"]
WARP_MODE = {"wreduce"}


def equivalence_sweep(seed: int = 20260823, per_kernel: int = 50) -> list:
    """test_acceptance.py:96-115: one RNG, 50 instances per kernel in order."""
    rng = random.Random(seed)
    out = []
    for name in EQUIVALENCE_CASES:
        for _ in range(per_kernel):
            out.append(CORPUS[name](rng))
    return out


# ---------------------------------------------------------------------------
# north-star generators (this repository's kernels/*.kn)
# ---------------------------------------------------------------------------

def f32(v: float) -> float:
    return struct.unpack("<f", struct.pack("<f", v))[0]


HOTSPOT_CONST = dict(  # Rodinia hotspot chip constants (double-valued params)
    t_chip=0.0005, chip_height=0.016, chip_width=0.016, amb=80.0)


def hotspot_params(rows: int, cols: int) -> dict:
    """Rodinia's derived constants step/Cap, 1/Rx, 1/Ry, 1/Rz (f64).

    The chip is scaled with the grid so the cell pitch stays Rodinia's
    1024x1024 pitch (0.016 m / 1024): with the 0.016 m chip an 8192^2 grid
    makes the explicit update unstable (step/Cap * 1/Ry = 8.7 > 1/4)."""
    max_pd, precision = 3.0e6, 0.001
    spec_heat_si, k_si, factor_chip = 1.75e6, 100.0, 0.5
    t_chip = HOTSPOT_CONST["t_chip"]
    h = HOTSPOT_CONST["chip_height"] * rows / 1024.0
    w = HOTSPOT_CONST["chip_width"] * cols / 1024.0
    grid_h = h / rows
    grid_w = w / cols
    cap = factor_chip * spec_heat_si * t_chip * grid_w * grid_h
    rx = grid_w / (2.0 * k_si * t_chip * grid_h)
    ry = grid_h / (2.0 * k_si * t_chip * grid_w)
    rz = t_chip / (k_si * grid_h * grid_w)
    max_slope = max_pd / (factor_chip * t_chip * spec_heat_si)
    step = precision / max_slope
    return dict(sdc=step / cap, rx1=1.0 / rx, ry1=1.0 / ry, rz1=1.0 / rz, amb=HOTSPOT_CONST["amb"])


def hotspot_inputs(rows: int, cols: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """temp ~ U(320, 340), power ~ U(0, 1e-3) from PCG64(seed), rounded to f32."""
    g = np.random.Generator(np.random.PCG64(seed))
    temp = g.uniform(320.0, 340.0, rows * cols).astype(np.float32)
    power = g.uniform(0.0, 1e-3, rows * cols).astype(np.float32)
    return temp, power


def hotspot(rows: int, cols: int, bx: int = 16, by: int = 16, seed: int = 0, gz: int = 1) -> Instance:
    temp, power = hotspot_inputs(rows, cols, seed)
    p = hotspot_params(rows, cols)
    gx, gy = -(-cols // bx), -(-rows // by)
    return Instance("hotspot", Geom(gx, gy, gz), Geom(bx, by), 0,
                    [Buf("src", "f32", rows * cols, temp), Buf("power", "f32", rows * cols, power),
                     Buf("dst", "f32", rows * cols, np.zeros(rows * cols, np.float32))],
                    [("buf", "src"), ("buf", "power"), ("buf", "dst"), ("i32", rows), ("i32", cols),
                     ("f32", p["sdc"]), ("f32", p["rx1"]), ("f32", p["ry1"]), ("f32", p["rz1"]),
                     ("f32", p["amb"])], ["dst"])


def nn_inputs(n: int, seed: int = 0) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(seed))
    ll = np.empty(2 * n, np.float32)
    ll[0::2] = g.uniform(-90.0, 90.0, n).astype(np.float32)
    ll[1::2] = g.uniform(-180.0, 180.0, n).astype(np.float32)
    return ll


NN_TARGET = (30.0, 90.0)  # Rodinia's default lat/lng query


def nn(n: int, block: int = 256, seed: int = 0, target=NN_TARGET) -> Instance:
    ll = nn_inputs(n, seed)
    gx = max(1, -(-n // block))
    return Instance("nn", Geom(gx), Geom(block), 0,
                    [Buf("ll", "f32", 2 * n, ll), Buf("d", "f32", max(n, 1), np.zeros(max(n, 1), np.float32))],
                    [("buf", "ll"), ("buf", "d"), ("i32", n), ("f32", target[0]), ("f32", target[1])],
                    ["d"])


def topk_distances(n: int, seed: int = 0, special: bool = False) -> np.ndarray:
    """Distance-like f32 values with many exact ties (one decimal); with
    `special`, also NaN, +inf, -0.0, 0.0 and negative values."""
    g = np.random.Generator(np.random.PCG64(seed))
    d = np.round(g.uniform(0.0, 50.0, n), 1).astype(np.float32)
    if special and n:
        picks = g.integers(0, n, size=min(n, 12))
        vals = [np.nan, np.inf, -0.0, 0.0, -1.5, np.nan, 0.0, -0.0, 3.0, -np.inf, np.nan, 0.1]
        for p, v in zip(picks, vals):
            d[p] = v
    return d


def nn_topk(n: int, k: int, seed: int = 0, special: bool = False, grid=(1,), block=(1,),
            idx_len=None, dist_len=None, d=None) -> Instance:
    d = topk_distances(n, seed, special) if d is None else np.asarray(d, np.float32)
    li = max(k, 1) if idx_len is None else idx_len
    ls = max(k, 1) if dist_len is None else dist_len
    return Instance("nn_topk", Geom(*grid), Geom(*block), 0,
                    [Buf("d", "f32", max(d.size, 1), d if d.size else np.zeros(1, np.float32)),
                     Buf("idx", "i32", li, np.full(li, 7, np.int32)),
                     Buf("dist", "f32", ls, np.full(ls, 9.0, np.float32))],
                    [("buf", "d"), ("buf", "idx"), ("buf", "dist"), ("i32", n), ("i32", k)],
                    ["idx", "dist"])


def kmeans_inputs(npts: int, nf: int, seed: int = 0) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(seed))
    return g.uniform(0.0, 1.0, npts * nf).astype(np.float32)  # feature-major f[l*npts + p]


def kmeans(npts: int, nf: int, k: int, block: int = 256, seed: int = 0, dup: bool = False) -> Instance:
    f = kmeans_inputs(npts, nf, seed)
    fm = f.reshape(nf, npts)
    cent = np.ascontiguousarray(fm[:, :k].T).reshape(-1)  # initial centroids = first k points
    if dup and k >= 2:  # force exact distance ties: cluster 1 duplicates cluster 0
        cent[nf:2 * nf] = cent[:nf]
    gx = max(1, -(-npts // block))
    return Instance("kmeans", Geom(gx), Geom(block), 0,
                    [Buf("f", "f32", npts * nf, f), Buf("cent", "f32", k * nf, cent),
                     Buf("member", "i32", npts, np.zeros(npts, np.int32)),
                     Buf("sums", "f32", k * nf, np.zeros(k * nf, np.float32)),
                     Buf("counts", "i32", k, np.zeros(k, np.int32))],
                    [("buf", "f"), ("buf", "cent"), ("buf", "member"), ("buf", "sums"), ("buf", "counts"),
                     ("i32", npts), ("i32", nf), ("i32", k)],
                    ["member", "sums", "counts"])


def random_graph(nv: int, deg: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """CSR of nv vertices x deg out-edges to uniform random targets (PCG64)."""
    g = np.random.Generator(np.random.PCG64(seed))
    col = g.integers(0, nv, size=nv * deg, dtype=np.int64).astype(np.int32)
    row = (np.arange(nv + 1, dtype=np.int64) * deg).astype(np.int32)
    return row, col


def bfs(nv: int, deg: int, cur: int = 0, seed: int = 0, block: int = 256, lvl=None) -> Instance:
    row, col = random_graph(nv, deg, seed)
    if lvl is None:
        lvl = np.full(nv, -1, np.int32)
        lvl[0] = 0
    gx = max(1, -(-nv // block))
    return Instance("bfs", Geom(gx), Geom(block), 0,
                    [Buf("row", "i32", nv + 1, row), Buf("col", "i32", len(col), col),
                     Buf("lvl", "i32", nv, np.asarray(lvl, np.int32)),
                     Buf("changed", "i32", 1, np.zeros(1, np.int32))],
                    [("buf", "row"), ("buf", "col"), ("buf", "lvl"), ("buf", "changed"), ("i32", nv),
                     ("i32", cur)], ["lvl", "changed"])


# ---- backprop (kernels/backprop.kn), Rodinia's 16 x 16 blocks, hid = 16 -----
BP_HID = 16


def backprop_forward(n_in: int, seed: int = 0, hid: int = BP_HID, block=(16, 16), grid_x: int = 1) -> Instance:
    """bpnn_layerforward over an input layer of n_in units (n_in % 16 == 0):
    grid 1 x n_in/16, weights U(0, 1) like bpnn_randomize_weights."""
    g = np.random.Generator(np.random.PCG64(seed))
    inp = g.uniform(0.0, 1.0, n_in + 1).astype(np.float32)
    w = g.uniform(0.0, 1.0, (n_in + 1) * (hid + 1)).astype(np.float32)
    nb = n_in // 16
    return Instance("bpnn_layerforward", Geom(grid_x, nb), Geom(*block), 0,
                    [Buf("input", "f32", n_in + 1, inp), Buf("w", "f32", w.size, w),
                     Buf("partial", "f32", nb * hid, np.zeros(nb * hid, np.float32))],
                    [("buf", "input"), ("buf", "w"), ("buf", "partial"), ("i32", hid)],
                    ["w", "partial"])


def backprop_adjust(n_in: int, seed: int = 0, hid: int = BP_HID, block=(16, 16)) -> Instance:
    """bpnn_adjust_weights of the input->hidden weights: delta (hid + 1),
    ly = input layer (n_in + 1), w / oldw (n_in + 1) x (hid + 1)."""
    g = np.random.Generator(np.random.PCG64(seed))
    delta = g.uniform(-0.1, 0.1, hid + 1).astype(np.float32)
    ly = g.uniform(0.0, 1.0, n_in + 1).astype(np.float32)
    w = g.uniform(0.0, 1.0, (n_in + 1) * (hid + 1)).astype(np.float32)
    oldw = g.uniform(-0.05, 0.05, (n_in + 1) * (hid + 1)).astype(np.float32)
    nb = n_in // 16
    return Instance("bpnn_adjust_weights", Geom(1, nb), Geom(*block), 0,
                    [Buf("delta", "f32", hid + 1, delta), Buf("ly", "f32", n_in + 1, ly),
                     Buf("w", "f32", w.size, w), Buf("oldw", "f32", oldw.size, oldw)],
                    [("buf", "delta"), ("i32", hid), ("buf", "ly"), ("i32", n_in), ("buf", "w"),
                     ("buf", "oldw")],
                    ["w", "oldw"])
