# kmeans_tg warp-role balance: 2 split sets + 1 epilogue set (480 threads) vs 1 + 2
for v in base s2e1 base s2e1; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans,kmeans_loop --steps 10 --warmup 3 > gpurun_out/tgs_$v.json 2>gpurun_out/tgs_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/tgs_$v.json').read().strip().splitlines()[-1]);print('$v', *[(n, k['ms_per_step'], k.get('checked')) for n, k in d['kernels'].items()])" 2>/dev/null || tail -2 gpurun_out/tgs_$v.err
done
cp alt_libs/s2e1.so paper_2206_07896_b200/libbfgpu.so
timeout 600 python -m pytest tests -m gpu -k kmeans -x -q 2>&1 | tail -2
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
