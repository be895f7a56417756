"""Which Python objects keep arenas alive after gpu_run? (memcheck leak triage)"""
import gc
import sys
sys.path[:0] = [".", "oracle", "tests"]
import instances as I
from gpu_helpers import gpu_run
from paper_2206_07896_b200 import DeviceArena, Runtime

inst = I.hotspot(64, 96, 16, 16, seed=5)
out = gpu_run(inst)
del out
live = [o for o in gc.get_objects() if isinstance(o, (DeviceArena, Runtime))]
print("live after gpu_run:", [type(o).__name__ for o in live])
for o in live:
    print(type(o).__name__, "referrers:", [type(r).__name__ for r in gc.get_referrers(o)][:8])
gc.collect()
print("live after gc:", [type(o).__name__ for o in gc.get_objects() if isinstance(o, (DeviceArena, Runtime))])
