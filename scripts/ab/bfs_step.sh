timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_jit.py tests/test_dropin.py -q -x -k "bfs or golden or pools" 2>&1 | tail -2
for v in 2 1; do
  BF_BFS_STEP_V=$v timeout 300 python bench.py --no-cpu --no-fused --cases bfs --steps 3 --warmup 2 > gpurun_out/bfsstep_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bfsstep_$v.json'));print('$v', d['kernels']['bfs']['ms_per_step'], d['kernels']['bfs']['checked'], d['kernels']['bfs'].get('levels'))"
done
