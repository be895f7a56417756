# kmeans_tc occupancy / ring depth variants (alt_libs built with -DKM_TC_MINB / -DKM_TC_STAGES)
for v in base m4s2 m3s2 m3s4 base m4s2; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 --iters 1 > gpurun_out/ko_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ko_$v.json'));print('$v', d['kernels']['kmeans']['ms_per_step'], d['kernels']['kmeans']['checked'])"
done
cp alt_libs/m4s2.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans" 2>&1 | tail -1
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
