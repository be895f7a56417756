# hotspot_band rows in flight (BF_HOTSPOT_PF)
for v in 1 2 3 4 1 2; do
  BF_HOTSPOT_PF=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/hpf_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hpf_$v.json'));print('pf', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'])"
done
