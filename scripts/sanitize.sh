# compute-sanitizer over the smoke run (every kernel family once, checked
# against the oracle) and the small-size parity tests: memcheck (out-of-bounds
# / misaligned global and shared accesses, leaks), racecheck (shared-memory
# hazards), synccheck (barrier misuse), initcheck (reads of uninitialised
# global memory).  Logs under gpurun_out/sanitize_*.log.
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 $CS --tool $tool $extra python -c "$SMOKE" > gpurun_out/sanitize_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
# small-size parity tests of the kernels with bulk copies / mbarriers / tcgen05 / RED
K="golden_sets or kmeans_vs_oracle_screen or bfs_levels_fused or bfs_transpose or hotspot_sizes or nn_vs_oracle or backprop_vs_oracle or hotspot_run_fused or topk"
for tool in memcheck racecheck synccheck; do
  timeout 2400 $CS --tool $tool python -m pytest tests/test_gpu_parity.py tests/test_nn_topk.py -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/sanitize_tests_$tool.log 2>&1
  echo "tests $tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
