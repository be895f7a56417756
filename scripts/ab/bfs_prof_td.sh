# ncu --set full of the top-down expansion at levels 7 and 8 and the bottom-up step at level 9 (2^26 x 8)
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:bfs_expand_v --launch-skip 7 --launch-count 2 -o gpurun_out/bfs_td python bench.py --no-cpu --no-fused --steps 1 --warmup 0 --cases bfs_do > gpurun_out/bfs_td.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:bfs_bottom_up --launch-skip 1 --launch-count 1 -o gpurun_out/bfs_bu2 python bench.py --no-cpu --no-fused --steps 1 --warmup 0 --cases bfs_do > gpurun_out/bfs_bu2.log 2>&1
