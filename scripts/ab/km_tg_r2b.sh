# kmeans_tg after the three-plane screen: ring-depth variants (alt_libs built
# with -D switches by scripts/altlib.py) and the per-tile trace of CTA 0
for v in base sa8 sp4st7 base sa8 sp4st7; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans,kmeans_loop --steps 10 --warmup 3 > gpurun_out/tgb_$v.json 2>gpurun_out/tgb_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/tgb_$v.json').read().strip().splitlines()[-1]);print('$v', *[(n, k['ms_per_step'], k.get('checked')) for n, k in d['kernels'].items()])" 2>/dev/null || tail -2 gpurun_out/tgb_$v.err
done
cp alt_libs/trace.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python scripts/micro/tg_trace.py > gpurun_out/tg_trace.log 2>&1; tail -14 gpurun_out/tg_trace.log
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
