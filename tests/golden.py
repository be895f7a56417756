"""Load tests/golden/*.npz (made by oracle/gen_golden.py from the reference
interpreter's own outputs) back into oracle.instances.Instance objects."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import instances as I

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str):
    """-> list of (instance, expected {buf: array}, trap kind or None)."""
    z = np.load(GOLDEN / f"{name}.npz")
    n = len([k for k in z.files if k.endswith("_meta")])
    replay = None
    if name == "corpus_sweep":
        replay = I.equivalence_sweep(20260823, 50)
    elif name == "corpus_extra":
        import random
        rng = random.Random(42)
        replay = [I.hist_stride(rng) for _ in range(30)]
        rng = random.Random(13)
        for _ in range(10):
            inst = I.wreduce(rng)
            inst.block = I.Geom(64)
            inst.grid = I.Geom(4)
            replay.append(inst)
    out = []
    for k in range(n):
        meta = json.loads(bytes(z[f"i{k}_meta"]).decode())
        if replay is not None:
            inst = replay[k]
            assert inst.kernel == meta["kernel"]
            assert [inst.grid.x, inst.grid.y, inst.grid.z] == meta["grid"]
        else:
            bufs = [I.Buf(bn, sc, ln, z[f"i{k}_in_{bn}"]) for bn, sc, ln in meta["buffers"]]
            inst = I.Instance(meta["kernel"], I.Geom(*meta["grid"]), I.Geom(*meta["block"]),
                              meta["shmem"], bufs, [tuple(a) for a in meta["args"]], meta["outputs"],
                              warp_size=meta["warp_size"])
        expected = {bn: z[f"i{k}_out_{bn}"] for bn, _, _ in meta["buffers"] if f"i{k}_out_{bn}" in z.files}
        out.append((inst, expected, meta["trap"]))
    return out


SETS = ["corpus_sweep", "corpus_extra", "geometry", "traps", "hotspot", "nn", "nn_topk", "kmeans", "bfs", "backprop"]
