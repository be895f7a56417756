# hotspot_band: alternating row direction (BF_HOTSPOT_ALT=1) vs top-down only
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hotspot or golden or full_size" 2>&1 | tail -1
for v in 1 0 1 0; do
  BF_HOTSPOT_ALT=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/ha_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ha_$v.json'));print('alt', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['e2e']['value'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hotspot_band -s 10 -c 4 --csv --log-file gpurun_out/hs_alt_ncu.csv python bench.py --no-cpu --no-kernels --no-fused --steps 1 --warmup 1 > /dev/null 2>&1
