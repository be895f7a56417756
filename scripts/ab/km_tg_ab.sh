# kmeans_tg variants (alt_libs built with -D switches), timing
for v in base st4 base st4; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  BF_KMEANS_V=5 timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/tga_$v.json 2>gpurun_out/tga_$v.err
  python -c "import json;d=json.load(open('gpurun_out/tga_$v.json'));k=d['kernels']['kmeans'];print('$v', k['ms_per_step'], k.get('checked'))" 2>/dev/null || tail -2 gpurun_out/tga_$v.err
done
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
