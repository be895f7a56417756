#!/bin/bash
for alt in 1 0; do
for v in ${VARIANTS:-7 6}; do
  BF_HOTSPOT_ALT=$alt BF_HOTSPOT_ROWS=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:hotspot_ -s 6 -c 4 --csv \
    python bench.py --steps 1 --warmup 3 --iters 10 --no-kernels --no-cpu --no-fused 2>/dev/null | grep -E '"(dram|gpu__time)' | awk -F'","' -v a=$alt -v v=$v '{print "alt="a, "v="v, $(NF-2), $NF}'
done
done
