# tcgen05 kmeans: parity (goldens + screen/ties/edge cases), bench, ncu
export BF_KMEANS_V=5
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans" 2>&1 | tail -15
timeout 240 python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 10 --warmup 3 > gpurun_out/km_v5.json 2>gpurun_out/km_v5.err
python -c "import json;d=json.load(open('gpurun_out/km_v5.json'));print(d['kernels']['kmeans'])"
tail -3 gpurun_out/km_v5.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:kmeans_umma -c 1 -o gpurun_out/kmeans_umma python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 1 --warmup 0 > /dev/null 2>&1
