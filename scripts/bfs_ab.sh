# fused BFS variants: parity of the new one, bench of each
BF_BFS_V=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs_levels_fused or full_size" 2>&1 | tail -1
for v in 2 3 4; do
  BF_BFS_V=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 2 > gpurun_out/bfs_v$v.json 2>gpurun_out/bfs_v$v.err
  python -c "import json;d=json.load(open('gpurun_out/bfs_v$v.json'));print('$v', d['kernels']['bfs_fused']['ms_per_step'], d['kernels']['bfs_fused']['checked'])"
done
