# per-level BFS launches: relax variants (BF_BFS_RELAX 0 claiming, 2 RED, 3 scan2 + RED + deferred dense lvl writes)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs or golden or traps or random" 2>&1 | tail -1
BF_BFS_DEFER_DIV=1000000 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs_levels_vs or golden" 2>&1 | tail -1
for v in 3 2 3 2; do
  BF_BFS_RELAX=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs --steps 5 --warmup 3 --iters 1 > gpurun_out/br_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/br_$v.json'));k=d['kernels']['bfs'];print('relax',$v,k['ms_per_step'],k['frac_hbm'],k['checked'])"
done
for dd in 16 256; do
  BF_BFS_DEFER_DIV=$dd timeout 300 python bench.py --no-cpu --no-fused --cases bfs --steps 5 --warmup 3 --iters 1 > gpurun_out/brd_$dd.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/brd_$dd.json'));k=d['kernels']['bfs'];print('div',$dd,k['ms_per_step'],k['frac_hbm'],k['checked'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_level_launches4.csv python bench.py --no-cpu --no-fused --cases bfs --steps 1 --warmup 0 --iters 1 > /dev/null 2>&1
