# nn_topk warp threshold + radix-sort transpose: parity, timings, then ncu captures
timeout 900 python -m pytest tests/test_nn_topk.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "topk or bfs" -p no:cacheprovider > gpurun_out/r2c4_tests.log 2>&1; tail -3 gpurun_out/r2c4_tests.log
timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases nn,nn_topk,bfs_do > gpurun_out/r2c4_bench.json 2> gpurun_out/r2c4_bench.err
bash scripts/r2_prof.sh
