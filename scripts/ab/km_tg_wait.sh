# kmeans_tg mbarrier wait styles (KM_TG_WAIT, alt_libs built by scripts/altlib.py)
for v in base w1 w2 w3 base w1 w2 w3; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans,kmeans_loop --steps 10 --warmup 3 > gpurun_out/tgw_$v.json 2>gpurun_out/tgw_$v.err
  python -c "import json;d=json.loads(open('gpurun_out/tgw_$v.json').read().strip().splitlines()[-1]);print('$v', *[(n, k['ms_per_step'], k.get('checked')) for n, k in d['kernels'].items()])" 2>/dev/null || tail -2 gpurun_out/tgw_$v.err
done
cp alt_libs/tracew3.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python scripts/micro/tg_trace.py > gpurun_out/tg_trace_w3.log 2>&1; tail -15 gpurun_out/tg_trace_w3.log | cut -c1-100
cp alt_libs/base.so paper_2206_07896_b200/libbfgpu.so
