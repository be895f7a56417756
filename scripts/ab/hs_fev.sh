# completion tracking: lazy cover events (BF_FETCH_EVENTS=2, default) vs one event per fetch (1)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hotspot or golden or full_size" 2>&1 | tail -1
for v in 1 0 1 0; do
  BF_FETCH_EVENTS=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/hf_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hf_$v.json'));print('fev', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['e2e']['value'])"
done
