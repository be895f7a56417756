timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hotspot_bands" -p no:cacheprovider > gpurun_out/r2c7_tests.log 2>&1; tail -3 gpurun_out/r2c7_tests.log
