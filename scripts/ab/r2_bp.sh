timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "backprop or golden" -p no:cacheprovider > gpurun_out/bp_tests.log 2>&1; tail -2 gpurun_out/bp_tests.log
timeout 600 python bench.py --no-cpu --no-fused --no-bfs --steps 5 --warmup 3 --cases bp_forward,bp_adjust > gpurun_out/bp_bench.json 2> gpurun_out/bp_bench.err
