# round 2 ncu --set full captures: hotspot_rows (headline), kmeans_tg, nn_topk_pass, bfs_tr (transpose)
mk() { timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 -c ${3:-1} -o gpurun_out/full_$2 python bench.py --no-cpu --no-fused --steps 1 --warmup 0 --cases $4 > gpurun_out/full_$2.log 2>&1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hotspot_rows --launch-skip 5 -c 1 -o gpurun_out/full_hotspot python bench.py --no-cpu --no-fused --no-kernels --steps 1 --warmup 0 > gpurun_out/full_hotspot.log 2>&1
mk kmeans_tg kmeans 1 kmeans
mk nn_topk_pass topk 1 nn,nn_topk
