for v in fir4 fir6 fir4 fir6; do
  cp alt_libs/$v.so paper_2206_07896_b200/libbfgpu.so
  timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases fir --steps 10 --warmup 3 > gpurun_out/f_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/f_$v.json'));print('$v', d['kernels']['fir']['ms_per_step'], d['kernels']['fir']['frac_hbm'], d['kernels']['fir']['checked'])"
done
