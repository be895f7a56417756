# fused BFS: pipelined host loop + coalesced compaction (default) vs the per-level loop
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs" 2>&1 | tail -1
BF_BFS_CS=0 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs_levels_fused" 2>&1 | tail -1
for cfg in "1 0" "0 0" "1 1" "1 0" "0 0"; do
  set -- $cfg
  BF_BFS_CS=$1 BF_BFS_APP=$2 timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused,bfs --steps 5 --warmup 3 --iters 1 > gpurun_out/bf3_$1_$2.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bf3_$1_$2.json'));k=d['kernels']['bfs_fused'];print('cs',$1,'app',$2,k['ms_per_step'],k['frac_hbm'],k['checked'], d['kernels']['bfs']['ms_per_step'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_fused_launches2.csv python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 --iters 1 > /dev/null 2>&1
