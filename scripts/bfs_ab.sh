# bucketed large BFS levels: parity, then A/B against the probing levels
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs_levels_fused or full_size or bfs_shards" 2>&1 | tail -2
for v in 1 0 1 0; do
  BF_BFS_BUCKET=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 2 > gpurun_out/bfsb_$v.json 2>gpurun_out/bfsb_$v.err
  python -c "import json;d=json.load(open('gpurun_out/bfsb_$v.json'));print('bucket $v', d['kernels']['bfs_fused']['ms_per_step'], d['kernels']['bfs_fused']['checked'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_launches3.csv python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 > /dev/null 2>&1
