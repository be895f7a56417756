# backprop on one GPU: parity tests, smoke, bench cases, ncu of both kernels
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "backprop or golden or pools" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu --no-fused --no-bfs --cases bp_forward,bp_adjust --steps 5 --warmup 3 > gpurun_out/bp.json 2>gpurun_out/bp.err
python -c "import json;d=json.load(open('gpurun_out/bp.json'));[print(k, d['kernels'][k]) for k in ('bp_forward','bp_adjust')]"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bp_ -c 2 -o gpurun_out/bp python bench.py --no-cpu --no-fused --no-bfs --cases bp_forward,bp_adjust --steps 1 --warmup 0 > /dev/null 2>&1
