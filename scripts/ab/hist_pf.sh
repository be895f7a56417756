# hist_range: software-pipelined loads (histpf) vs base
for v in histpf base histpf base; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases hist,hist_stride --steps 10 --warmup 3 --iters 1 > gpurun_out/hp_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hp_$v.json'));k=d['kernels'];print('$v', k['hist']['ms_per_step'], k['hist']['frac_hbm'], k['hist_stride']['frac_hbm'], k['hist']['checked'])"
done
cp alt_libs/histpf.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "hist or golden" 2>&1 | tail -1
