timeout 900 python -m pytest tests/test_nn_topk.py tests/test_gpu_parity.py -m gpu -q -x -k "topk or golden" -p no:cacheprovider > gpurun_out/r2c8_tests.log 2>&1; tail -3 gpurun_out/r2c8_tests.log
timeout 600 python bench.py --no-cpu --no-fused --no-bfs --steps 5 --warmup 3 --cases nn,nn_topk > gpurun_out/r2c8_bench.json 2> gpurun_out/r2c8_bench.err
