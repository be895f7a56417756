timeout 600 python bench.py --no-cpu --no-fused --no-bfs --steps 5 --warmup 3 --cases nn,nn_topk > gpurun_out/r2c9_bench.json 2> gpurun_out/r2c9_bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:nn_topk_pass -c 1 -o gpurun_out/full_topk2 python bench.py --no-cpu --no-fused --no-bfs --steps 1 --warmup 0 --cases nn,nn_topk > /dev/null 2>&1
