# kmeans_tg ring-depth variants (alt_libs built with -DKM_TG_ST / -DKM_TG_SP), timing + the variant parity test
for v in base st4 s6t4 s6t5 s6t6 base; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  BF_KMEANS_V=5 timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/tga_$v.json 2>gpurun_out/tga_$v.err
  python -c "import json;d=json.load(open('gpurun_out/tga_$v.json'));k=d['kernels']['kmeans'];print('$v', k['ms_per_step'], k.get('checked'))" || tail -3 gpurun_out/tga_$v.err
done
for v in s6t4 base; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  BF_KMEANS_V=5 timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "kmeans" 2>&1 | tail -1
done
