for v in 0 1 0 1; do
  BF_HOTSPOT_STCS=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/hs_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hs_$v.json'));print('stcs', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'])"
done
