# round-2 check: new full-size / partial-fetch parity tests, bench contract, default bench
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_bench_contract.py -x -q > gpurun_out/fullsize.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/fullsize.log
