# full round check on one B200: smoke, GPU tests, default bench, ncu launch list,
# and the kmeans_tg ncu --set full capture
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kmeans_tg -c 1 -o gpurun_out/full_kmeans -f python bench.py --no-cpu --no-fused --no-bfs --steps 1 --warmup 0 --cases kmeans > gpurun_out/full_kmeans.log 2>&1
tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/gputests.log
