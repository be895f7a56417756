# compute-sanitizer on kmeans_tg (memcheck, synccheck, racecheck) + the kmeans variant tests
for tool in memcheck synccheck racecheck; do
  timeout 600 compute-sanitizer --tool $tool --show-backtrace no --kernel-name kns=kmeans_tg python scripts/micro/tg_sanitize.py > gpurun_out/tg_san_$tool.log 2>&1
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|member equal|Error" gpurun_out/tg_san_$tool.log | head -5
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kmeans_variants" 2>&1 | tail -1
