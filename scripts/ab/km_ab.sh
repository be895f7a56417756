# kmeans tensor-core variants on one GPU (alt_libs/*.so swapped in turn)
for v in m3 m4; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/km_$v.json 2>gpurun_out/km_$v.err
  python -c "import json;d=json.load(open('gpurun_out/km_$v.json'));print('$v', d['kernels']['kmeans']['ms_per_step'], d['kernels']['kmeans']['frac_hbm'])"
done
cp alt_libs/m3.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans" 2>&1 | tail -2
