# round 2: device-fetch / nn_topk / runtime parity, grain study (host vs device fetching), smoke under memcheck
timeout 1200 python -m pytest tests/test_device_fetch.py tests/test_nn_topk.py tests/test_runtime.py tests/test_jit.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2c2_tests.log 2>&1; tail -5 gpurun_out/r2c2_tests.log
timeout 900 python bench.py --workload grain > gpurun_out/r2c2_grain.json 2> gpurun_out/r2c2_grain.err
timeout 900 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r2c2_memcheck.log 2>&1; tail -3 gpurun_out/r2c2_memcheck.log
