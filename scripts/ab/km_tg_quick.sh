# kmeans_tg quick check: sums/membership debug script + timing + trace
timeout 200 python scripts/micro/tg_sums_dbg.py 2>&1 | tail -6
BF_KMEANS_V=5 timeout 200 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/tgq.json 2>gpurun_out/tgq.err
python -c "import json;d=json.load(open('gpurun_out/tgq.json'));k=d['kernels']['kmeans'];print('tg', k['ms_per_step'], k.get('checked'))" 2>/dev/null || tail -2 gpurun_out/tgq.err
cp alt_libs/trace.so paper_2206_07896_b200/libbfgpu.so
timeout 200 python scripts/micro/tg_trace.py 2>&1 | tail -12
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
