# per-launch durations and L2 / DRAM metrics of one fused BFS traversal (2^26 x 8)
timeout 900 ncu --metrics gpu__time_duration.sum,lts__t_sectors.sum,dram__bytes_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:bfs_ --csv --log-file gpurun_out/bfs_fused_launches.csv python bench.py --no-cpu --no-fused --cases bfs_fused --steps 1 --warmup 0 --iters 1 > gpurun_out/bfs_prof2.log 2>&1
tail -3 gpurun_out/bfs_prof2.log
