# round 2: tcgen05 layout probe, kmeans_t5 / device-fetch / nn_topk parity, kernel timings, grain study
./scripts/micro/umma_sw128 > gpurun_out/umma_sw128.log 2>&1; tail -12 gpurun_out/umma_sw128.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_device_fetch.py tests/test_nn_topk.py tests/test_runtime.py -m gpu -q -x -k "kmeans or fetch or topk or grains or every_block" -p no:cacheprovider > gpurun_out/r2c1_tests.log 2>&1; tail -15 gpurun_out/r2c1_tests.log
timeout 600 python bench.py --no-cpu --no-fused --no-bfs --steps 5 --warmup 3 --cases kmeans,kmeans_loop,nn_topk,vecadd > gpurun_out/r2c1_bench.json 2> gpurun_out/r2c1_bench.err
timeout 900 python bench.py --workload grain > gpurun_out/r2c1_grain.json 2> gpurun_out/r2c1_grain.err
