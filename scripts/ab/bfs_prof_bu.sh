# ncu --set full of the bottom-up step (alpha16=64: bottom-up from level 8 on)
BF_BFS_ALPHA16=64 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:bfs_bottom_up -c 4 -o gpurun_out/bfs_bu python bench.py --no-cpu --no-fused --steps 1 --warmup 0 --cases bfs_do > gpurun_out/bfs_bu.log 2>&1
tail -3 gpurun_out/bfs_bu.log
