run() {
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o gpurun_out/full_$1 python bench.py --no-cpu --no-fused --steps 1 --warmup 1 --iters 1 $4 > /dev/null 2>&1
}
run hist 'hist_range' 1 "--no-bfs --cases hist"
run nn 'nn_stream' 1 "--no-bfs --cases nn"
run kmeans 'kmeans_tc' 1 "--no-bfs --cases kmeans"
ls -la gpurun_out/full_*.ncu-rep
