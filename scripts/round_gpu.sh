# full round check on one B200: smoke, GPU tests, default bench, ncu launch list
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu --steps 2 --warmup 1 > /dev/null 2>&1
tail -1 gpurun_out/smoke.log; tail -2 gpurun_out/gputests.log
