# per-kernel ncu captures of the streaming corpus kernels + their bench lines
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "large_random or golden or random_instances" 2>&1 | tail -1
timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases fir,hist,reduce,hist_stride --steps 5 --warmup 3 > gpurun_out/corpus.json 2>gpurun_out/corpus.err
python -c "import json;d=json.load(open('gpurun_out/corpus.json'));[print(k, v['ms_per_step'], v['frac_hbm']) for k,v in d['kernels'].items()]"
for k in fir_reg hist_range reduce_warp; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/prof_$k python bench.py --no-cpu --no-fused --no-bfs --cases fir,hist,reduce --steps 1 --warmup 0 > /dev/null 2>&1
done
