"""Per-tile timeline of kmeans_tg's CTA 0 (alt_libs/trace.so built with -DKM_TG_TRACE)."""
import ctypes, os, sys
import numpy as np
sys.path[:0] = [os.getcwd(), os.getcwd() + "/oracle", os.getcwd() + "/tests"]
os.environ["BF_KMEANS_V"] = "5"
import instances as I
from gpu_helpers import gpu_run
import paper_2206_07896_b200._lib as L
inst = I.kmeans(1 << 24, 32, 16, 256, seed=0)
for _ in range(2):
    gpu_run(inst)
buf = (ctypes.c_ulonglong * (12 * 2048))()
lib = ctypes.CDLL(os.path.join(os.getcwd(), "paper_2206_07896_b200/libbfgpu.so"))
print("rc", lib.bf_debug_tg_trace(buf))
t = np.frombuffer(buf, dtype=np.uint64).reshape(12, 2048).astype(np.int64)
n = int((t[0] > 0).sum())
t = t[:, :n] - t[0, 0]
names = ["tma_issue", "split_got_tile", "split_got_planes", "split_done", "dist_issued", "epi_got_acc", "epi_done",
         "sums_issued", "mma_got_full_p", "mma_got_acc_empty", "mma_got_oh_full", "split_released"]
base = t[0, n // 2]
short = ["tma", "s_tile", "s_pl", "s_done", "d_iss", "e_acc", "e_done", "sum_iss", "m_fp", "m_ae", "m_oh", "s_rel"]
for i in list(range(n // 2, n // 2 + 10)):
    print(i, " ".join(f"{short[e]}={(t[e, i] - base) if t[e, i] > 0 else -1:6d}" for e in range(12)))  # cycles
d = np.diff(t[6, 10:n - 10])
print("tiles", n, "median epi_done interval (cycles)", np.median(d))
rel, iss = t[11, 10:n - 15], t[0, 15:n - 10]
print(f"split_released(n) -> tma_issue(n + 5): median {np.median(iss - rel):.0f} cycles")
for a, b in [(0, 1), (1, 2), (2, 11), (2, 3), (3, 8), (8, 9), (9, 4), (4, 5), (5, 6), (6, 10), (10, 7), (0, 6)]:
    print(f"{names[a]} -> {names[b]}: median {np.median(t[b, 10:n-10] - t[a, 10:n-10]):.0f} cycles")
