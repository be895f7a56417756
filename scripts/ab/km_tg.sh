# kmeans_tg (BF_KMEANS_V=5) vs kmeans_tc (4): parity (variant + full-size tests), timing x3
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kmeans_variants and 5" > gpurun_out/tg_var.log 2>&1
tail -1 gpurun_out/tg_var.log
BF_KMEANS_V=5 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -m gpu -q -x -k "kmeans" > gpurun_out/tg_full.log 2>&1
tail -1 gpurun_out/tg_full.log
for v in 4 5 5 5; do
  BF_KMEANS_V=$v timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans,kmeans_loop --steps 10 --warmup 3 > gpurun_out/tg_$v.json 2>gpurun_out/tg_$v.err
  python -c "import json;d=json.load(open('gpurun_out/tg_$v.json'));k=d['kernels'];print('$v', k['kmeans']['ms_per_step'], k['kmeans'].get('checked'), k['kmeans_loop']['ms_per_step'])" 2>/dev/null || tail -2 gpurun_out/tg_$v.err
done
cp alt_libs/trace.so paper_2206_07896_b200/libbfgpu.so
timeout 200 python scripts/micro/tg_trace.py 2>&1 | tail -12
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
