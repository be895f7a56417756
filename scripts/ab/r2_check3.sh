# round 2 check on HEAD: smoke, every GPU test, default bench, launch list; leak triage; bfs_do timing
python scripts/micro/leak_probe.py > gpurun_out/leak_probe.log 2>&1
bash scripts/round_gpu.sh
timeout 600 python bench.py --no-cpu --no-fused --steps 5 --warmup 3 --cases bfs_fused,bfs_do,nn_topk > gpurun_out/r2c3_bfs.json 2> gpurun_out/r2c3_bfs.err
