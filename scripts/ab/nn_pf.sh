# nn_stream: software-pipelined loads (nnpf) vs base
for v in nnpf base nnpf base; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases nn --steps 10 --warmup 3 --iters 1 > gpurun_out/np_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/np_$v.json'));k=d['kernels'];print('$v', k['nn']['ms_per_step'], k['nn']['frac_hbm'], k['nn']['checked'])"
done
cp alt_libs/nnpf.so paper_2206_07896_b200/libbfgpu.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "nn or golden" 2>&1 | tail -1
