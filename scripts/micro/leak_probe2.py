"""Device memory before / after an arena + runtime lifetime (memcheck leak triage)."""
import gc
import sys
sys.path[:0] = [".", "oracle", "tests"]
import torch
import instances as I
from gpu_helpers import gpu_run

torch.cuda.init()
def used():
    f, t = torch.cuda.mem_get_info()
    return (t - f) >> 20
inst = I.hotspot(256, 512, 16, 16, seed=5)
gpu_run(inst)
gc.collect()
u0 = used()
for _ in range(5):
    out = gpu_run(inst)
    del out
gc.collect()
print("device MiB used before / after 5 gpu_run:", u0, used(), flush=True)
from paper_2206_07896_b200 import DeviceArena, Runtime
live = [o for o in gc.get_objects() if isinstance(o, (DeviceArena, Runtime))]
print("live:", [type(o).__name__ for o in live], flush=True)
for o in live[:2]:
    for r in gc.get_referrers(o)[:6]:
        print("  referrer of", type(o).__name__, ":", type(r).__name__, str(r)[:200], flush=True)
