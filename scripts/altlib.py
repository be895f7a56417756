import subprocess, sys
sys.path.insert(0, '/root/repo')
from paper_2206_07896_b200 import build as B
name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
objs = [B.BUILD / (s.stem + ".o") for s in B.sources()]
alt = B.BUILD / f"alt_{name}.o"
subprocess.run([B.nvcc()] + B.NVCC_FLAGS + defs + ["-c", str(B.CSRC / src), "-o", str(alt)], check=True)
objs = [alt if o.stem == src[:-3] else o for o in objs]
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", f"/root/repo/alt_libs/{name}.so"] + [str(o) for o in objs] +
               ["-lcudart_static", "-lrt", "-ldl", "-lpthread", "-L/usr/local/cuda/lib64", "-lnvrtc", "-Xlinker", "-rpath,/usr/local/cuda/lib64"], check=True)
print("ok", name)
