# one ncu --set full capture per kernel of interest (round-1 summary table)
run() {  # name, kernel regex, skip, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s $3 -c 1 -f -o gpurun_out/full_$1 python bench.py --no-cpu --no-fused --steps 1 --warmup 1 --iters 1 $4 > /dev/null 2>&1
}
run hotspot_band 'hotspot_band' 5 "--no-kernels"
run hist 'hist_range' 2 "--no-bfs --cases hist"
run nn 'nn_stream' 2 "--no-bfs --cases nn"
run relax 'bfs_relax_v' 9 "--cases bfs"
run compact8s 'bfs_compact8s' 9 "--cases bfs_fused"
run expand 'bfs_expand_v' 9 "--cases bfs_fused"
ls -la gpurun_out/full_*.ncu-rep
