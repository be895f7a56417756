timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sharded or views or bfs_shards" > gpurun_out/shard.log 2>&1
timeout 600 python -m pytest tests/test_bench_contract.py -x -q >> gpurun_out/shard.log 2>&1
timeout 600 python bench.py --workload kmeans --steps 3 --warmup 3 > gpurun_out/kmeans_loop.json 2>gpurun_out/kmeans_loop.err
tail -3 gpurun_out/shard.log
