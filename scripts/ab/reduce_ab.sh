for v in 0 1 2 3; do
  BF_REDUCE_V=$v timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases reduce --steps 10 --warmup 3 > gpurun_out/red_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/red_$v.json'));print($v, d['kernels']['reduce']['ms_per_step'], d['kernels']['reduce']['frac_hbm'], d['kernels']['reduce']['checked'])"
done
