# launch list of the direction-optimizing traversal (per-level kernel times, DRAM bytes, L2 sectors)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum --clock-control none --csv -k regex:bfs --log-file gpurun_out/bfs_do_launches.csv python bench.py --no-cpu --no-fused --steps 1 --warmup 1 --cases bfs_do > /dev/null 2>&1
