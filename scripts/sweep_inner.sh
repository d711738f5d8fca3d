#!/bin/bash
for k in 1 2 4 8 16 64; do
  echo "== KNF_MARCH_MAX_INNER=$k"
  KNF_MARCH_MAX_INNER=$k python scripts/gpu_probe.py 2>&1 | grep -E "render .* (800x800|1920x1080)"
done
