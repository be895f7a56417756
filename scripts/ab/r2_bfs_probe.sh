for p in 1 0 2; do BF_BFS_PROBE=$p timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases bfs_fused,bfs_do > gpurun_out/probe_$p.json 2>/dev/null; done
BF_BFS_PROBE=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bfs_levels_fused or bfs_opt_in" -p no:cacheprovider > gpurun_out/probe_tests.log 2>&1; tail -2 gpurun_out/probe_tests.log
