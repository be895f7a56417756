timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "bfs" -p no:cacheprovider > gpurun_out/r2c10_tests.log 2>&1; tail -2 gpurun_out/r2c10_tests.log
timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases bfs,bfs_do > gpurun_out/r2c10_bench.json 2> gpurun_out/r2c10_bench.err
