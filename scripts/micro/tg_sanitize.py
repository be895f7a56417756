"""Two small kmeans launches (kmeans_tg) for compute-sanitizer runs."""
import os
import sys
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
import numpy as np
import instances as I
import oracle
from gpu_helpers import gpu_run
for inst in (I.kmeans(128 * 148 * 2 + 36, 32, 16, 256, seed=5, dup=True), I.kmeans(4096, 32, 5, 256, seed=6)):
    want, _ = oracle.run(inst)
    got, trap, _, _ = gpu_run(inst)
    print("member equal", np.array_equal(got["member"], want["member"]), "trap", trap)
