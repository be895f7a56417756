import os, sys
import numpy as np
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
os.environ.setdefault("BF_KMEANS_V", "5")
import instances as I
import oracle
from gpu_helpers import gpu_run
from paper_2206_07896_b200 import Fixed
for npts, pool, pol in [(128 * 148, 1, None), (256 * 148, 1, None), (384 * 148, 1, None), (1 << 16, 1, None), (1 << 16, 2, None), (1 << 18, 2, None)]:
    inst = I.kmeans(npts, 32, 16, 256, seed=3)
    want, _ = oracle.run(inst, nthreads=8)
    got, trap, _, _ = gpu_run(inst, pool_size=pool)
    w, g = want["sums"].astype(np.float64), got["sums"].astype(np.float64)
    print(npts, pool, "member ok", np.array_equal(got["member"], want["member"]), "counts ok", np.array_equal(got["counts"], want["counts"]),
          "sums max rel", np.max(np.abs(w - g) / np.maximum(np.abs(w), 1)), "ratio", (g.sum() / w.sum()))
