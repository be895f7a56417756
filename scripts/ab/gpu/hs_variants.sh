#!/bin/bash
# hotspot kernel variants: parity then per-variant bench line (BF_HOTSPOT_ROWS)
mkdir -p gpurun_out
for v in ${VARIANTS:-1 0 2 3 4}; do
  echo "== variant $v"
  BF_HOTSPOT_ROWS=$v timeout 300 python -m pytest tests -m gpu -x -q -k "hotspot" 2>&1 | tail -2
  BF_HOTSPOT_ROWS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-kernels --no-cpu --no-fused > gpurun_out/hs_v$v.json 2> gpurun_out/hs_v$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/hs_v{v}.json").read().strip().splitlines()[-1])
    print(v, d["value"], d["roofline"]["frac"], d["roofline"]["avg_launch_us"], d["e2e"]["value"], d["clocks"]["sm_mhz"])
except Exception as e:
    print(v, "failed", e, open(f"gpurun_out/hs_v{v}.err").read()[-2000:])
PY
done
