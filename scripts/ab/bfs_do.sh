# direction-optimizing BFS: parity tests, alpha sweep of the fused traversal at 2^26 x 8
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "bfs" > gpurun_out/bfs_tests.log 2>&1
tail -3 gpurun_out/bfs_tests.log
for a in 16 32 64 96; do
  BF_BFS_ALPHA16=$a timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases bfs_fused,bfs_do > gpurun_out/bfs_a$a.json 2> gpurun_out/bfs_a$a.err
done
python - <<'PY'
import json
for a in (16,32,64,96):
    try:
        d=json.loads(open(f'gpurun_out/bfs_a{a}.json').read().strip().splitlines()[-1])
        k=d['kernels']; print(a, {n:(k[n]['ms_per_step'],k[n].get('checked'),k[n].get('transpose_build_ms')) for n in k})
    except Exception as e: print(a, e)
PY
