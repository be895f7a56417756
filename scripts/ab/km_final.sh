# kmeans parity after the last kmeans_tg changes + the kmeans workload line (with e2e)
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kmeans" > gpurun_out/kf_par.log 2>&1; tail -1 gpurun_out/kf_par.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "kmeans" > gpurun_out/kf_full.log 2>&1; tail -1 gpurun_out/kf_full.log
timeout 600 python bench.py --workload kmeans --steps 3 --warmup 1 > gpurun_out/kf_bench.json 2> gpurun_out/kf_bench.err; tail -1 gpurun_out/kf_bench.json; tail -2 gpurun_out/kf_bench.err
