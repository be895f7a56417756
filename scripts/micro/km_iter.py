import sys
sys.path[:0] = ['/root/repo', '/root/repo/oracle', '/root/repo/tests']
import numpy as np
import instances as I
from paper_2206_07896_b200 import DeviceArena, Runtime
from paper_2206_07896_b200.cluster import KmeansDriver
npts, nf, k = 50000, 32, 16
fv = I.kmeans_inputs(npts, nf, seed=33)
for rep in range(3):
    arena = DeviceArena()
    hf, hc, hm = arena.alloc("f32", npts * nf), arena.alloc("f32", k * nf), arena.alloc("i32", npts)
    arena.upload_numpy(hf, fv)
    arena.upload_numpy(hc, np.ascontiguousarray(fv.reshape(nf, npts)[:, :k].T).reshape(-1))
    with Runtime(arena) as rt:
        drv = KmeansDriver(rt, arena, hf, hc, hm, npts, nf, k, 1, 0)
        ds = []
        for p in range(300):
            drv.assign(); d = drv.update(); ds.append(d)
            if d == 0: break
        print(rep, len(ds), ds[:8], ds[-12:])
