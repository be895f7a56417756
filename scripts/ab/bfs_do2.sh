# direction-optimizing BFS with append-mode small levels: parity tests, small_div sweep
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "bfs" > gpurun_out/bfs_tests.log 2>&1
tail -3 gpurun_out/bfs_tests.log
for dv in 0 256 1024 4096; do
  BF_BFS_SMALL_DIV=$dv timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases bfs_fused,bfs_do > gpurun_out/bfs_d$dv.json 2> gpurun_out/bfs_d$dv.err
done
