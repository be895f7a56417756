timeout 900 python -m pytest tests/test_device_fetch.py tests/test_runtime.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2c11_tests.log 2>&1; tail -2 gpurun_out/r2c11_tests.log
timeout 900 python bench.py --workload grain > gpurun_out/r2c11_grain.json 2> gpurun_out/r2c11_grain.err
