"""H2D / D2H bandwidth alone and concurrent (two streams, pinned host memory)."""
import time
import torch
d = torch.device("cuda", 0)
a_h = torch.empty(128 << 20, dtype=torch.float32).pin_memory()   # 512 MB
b_h = torch.empty(64 << 20, dtype=torch.float32).pin_memory()    # 256 MB
a_d = torch.empty_like(a_h, device=d)
b_d = torch.empty_like(b_h, device=d)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def h2d():
    with torch.cuda.stream(s1): a_d.copy_(a_h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): b_h.copy_(b_d, non_blocking=True)
for name, fns in [("h2d 512MB", [h2d]), ("d2h 256MB", [d2h]), ("both", [h2d, d2h])]:
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for f in fns: f()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{name}: {dt*1e3:.2f} ms", flush=True)
