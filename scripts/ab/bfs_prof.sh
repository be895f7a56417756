# fused BFS launch list with per-launch DRAM and L2 metrics
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_launches.csv python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 > gpurun_out/bfs_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bfs_expand --launch-skip 8 -c 1 -o gpurun_out/bfs_expand python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 > /dev/null 2>&1
tail -2 gpurun_out/bfs_prof.log
