# fused + per-level BFS after the CTA-level queue appends: parity and timing
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs or full_size" 2>&1 | tail -1
timeout 300 python bench.py --no-cpu --no-fused --cases bfs,bfs_fused --steps 5 --warmup 2 > gpurun_out/bfs_new.json 2>gpurun_out/bfs_new.err
python -c "import json;d=json.load(open('gpurun_out/bfs_new.json'));[print(k, d['kernels'][k]['ms_per_step'], d['kernels'][k]['checked']) for k in ('bfs','bfs_fused')]"
