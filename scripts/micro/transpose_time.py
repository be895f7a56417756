"""Time bf_bfs_transpose on the 2^26 x 8 bench graph (wall, 3 calls)."""
import sys
import time
sys.path[:0] = ["."]
import torch
from paper_2206_07896_b200 import DeviceArena, Runtime, graph

nv, deg = 1 << 26, 8
arena = DeviceArena(0)
row, col = arena.alloc("i32", nv + 1), arena.alloc("i32", nv * deg)
dev = torch.device("cuda", 0)
torch.as_tensor(arena.cuda_array(row), device=dev).copy_(torch.arange(0, nv + 1, dtype=torch.int64, device=dev).mul_(deg).int())
torch.as_tensor(arena.cuda_array(col), device=dev).random_(0, nv)
torch.cuda.synchronize()
with Runtime(arena) as rt:
    for i in range(3):
        t0 = time.perf_counter()
        tg = graph.transpose(rt, row, col, nv)
        torch.cuda.synchronize()
        print(f"transpose {i}: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
        arena.free(tg.crow)
        arena.free(tg.ccol)
