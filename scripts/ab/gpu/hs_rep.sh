#!/bin/bash
for rep in 1 2 3; do
for v in ${VARIANTS:-6 9}; do
  BF_HOTSPOT_ROWS=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-kernels --no-cpu --no-fused > gpurun_out/hs_ev.json 2>gpurun_out/hs_ev.err
  python3 -c "
import json; d=json.loads(open('gpurun_out/hs_ev.json').read().strip().splitlines()[-1]); print('rep $rep v=$v', d['value'], d['roofline']['avg_launch_us'], d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/hs_ev.err
done
done
