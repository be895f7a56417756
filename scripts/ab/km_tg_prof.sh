BF_KMEANS_V=5 timeout 600 ncu --set full --import-source on --clock-control none -k regex:kmeans_tg -c 1 -o gpurun_out/kmeans_tg -f python bench.py --no-cpu --no-fused --no-bfs --cases kmeans --steps 1 --warmup 1 > gpurun_out/tg_ncu.log 2>&1
tail -2 gpurun_out/tg_ncu.log
