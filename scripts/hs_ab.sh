# hotspot per-launch variants (register prefetch vs cp.async ring depths)
for v in 0 3 4 6 8; do
  BF_HOTSPOT_RING=$v timeout 300 python bench.py --no-cpu --no-kernels --no-fused --steps 5 --warmup 3 > gpurun_out/hs_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hs_$v.json'));print('ring', $v, d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'])"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kmeans_tc -c 1 -o gpurun_out/kmeans_tc2 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 1 --warmup 0 > /dev/null 2>&1
