#!/bin/bash
mkdir -p gpurun_out
for v in ${VARIANTS:-1}; do
  BF_HOTSPOT_ROWS=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:hotspot_ -s 5 -c 1 \
    -o gpurun_out/hs_v$v -f python bench.py --steps 1 --warmup 3 --iters 10 --no-kernels --no-cpu --no-fused > gpurun_out/hs_ncu_v$v.log 2>&1
  tail -1 gpurun_out/hs_ncu_v$v.log
done
