#!/bin/bash
for v in ${VARIANTS:-7}; do
for ev in "" "--launch-events"; do
  BF_HOTSPOT_ROWS=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-kernels --no-cpu --no-fused $ev > gpurun_out/hs_ev.json 2>gpurun_out/hs_ev.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/hs_ev.json').read().strip().splitlines()[-1]); print('$v', '$ev', d['value'], d['ms_per_step'], d['roofline']['avg_launch_us'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/hs_ev.err
done
done
