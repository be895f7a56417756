# fused BFS: compaction with prefetched words and empty-iteration skip (c2) vs base
for v in c2 base c2 base; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 300 python bench.py --no-cpu --no-fused --cases bfs_fused --steps 5 --warmup 3 --iters 1 > gpurun_out/bc2_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bc2_$v.json'));k=d['kernels'];print('$v', k['bfs_fused']['ms_per_step'], k['bfs_fused']['checked'])"
done
cp alt_libs/c2.so paper_2206_07896_b200/libbfgpu.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "bfs" 2>&1 | tail -1
