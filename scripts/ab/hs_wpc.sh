# hotspot_band warps per CTA: 4 / 8 / 16
BF_HOTSPOT_WPC=16 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "hotspot" 2>&1 | tail -1
for v in 4 8 16 4 8 16; do
  BF_HOTSPOT_WPC=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/hw_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hw_$v.json'));print('wpc', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['e2e']['value'])"
done
