for v in u23 u32; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  BF_KMEANS_V=5 timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/km_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/km_$v.json'));print('$v', d['kernels']['kmeans']['ms_per_step'], d['kernels']['kmeans']['checked'])"
done
BF_KMEANS_V=5 timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans" 2>&1 | tail -1
