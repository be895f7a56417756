timeout 600 python scripts/micro/transpose_time.py > gpurun_out/transpose_time.log 2>&1; cat gpurun_out/transpose_time.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"bfs_tr|Radix|radix|Onesweep|onesweep|Histogram|histogram|Exclusive" --log-file gpurun_out/transpose_launches.csv python scripts/micro/transpose_time.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_nn_topk.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2c5_tests.log 2>&1; tail -2 gpurun_out/r2c5_tests.log
timeout 600 python bench.py --no-cpu --no-fused --no-bfs --steps 5 --warmup 3 --cases nn,nn_topk > gpurun_out/r2c5_bench.json 2> gpurun_out/r2c5_bench.err
