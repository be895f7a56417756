#!/bin/bash
BF_HOTSPOT_ROWS=7 timeout 300 python -m pytest tests -m gpu -x -q -k "hotspot" 2>&1 | tail -2
for alt in 1 0; do
  BF_HOTSPOT_ALT=$alt VARIANTS="7 6" bash scripts/gpu/hs_events.sh | grep step-events | sed "s/^/alt=$alt /"
done
