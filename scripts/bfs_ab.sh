# fused BFS variants: parity under each, bench, per-launch list of the new variant
for v in 3; do
  BF_BFS_V=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs" 2>&1 | tail -1
  BF_BFS_V=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 2 --no-kernels > /dev/null 2>&1
  BF_BFS_V=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 2 > gpurun_out/bfs_v$v.json 2>gpurun_out/bfs_v$v.err
  python -c "import json;d=json.load(open('gpurun_out/bfs_v$v.json'));print('$v', d['kernels']['bfs_fused'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_launches2.csv python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 > /dev/null 2>&1
