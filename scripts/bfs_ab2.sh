# fused BFS: coalesced compaction (BF_BFS_CS) and fused append for small levels (BF_BFS_APP)
BF_BFS_APP=256 BF_BFS_CS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs" 2>&1 | tail -1
BF_BFS_APP=16 BF_BFS_CS=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs_levels_fused" 2>&1 | tail -1
for cfg in "0 0" "0 1" "256 1" "64 1" "1024 1" "0 0" "256 1"; do
  set -- $cfg
  BF_BFS_APP=$1 BF_BFS_CS=$2 timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 3 --iters 1 > gpurun_out/bf2_$1_$2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bf2_$1_$2.json'));k=d['kernels']['bfs_fused'];print('app',$1,'cs',$2,k['ms_per_step'],k['frac_hbm'],k['checked'])"
done
