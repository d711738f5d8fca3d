#!/bin/bash
# A/B the tile-kernel variants built as libknf_w{1,2,4}.so
for w in 1 2 4; do
  echo "== KNF_TILE_WARPS=$w"
  KNF_B200_LIB=$PWD/paper_2206_10885_b200/libknf_w$w.so python scripts/gpu_probe.py 2>&1 | grep -E "sdf_query M=|render .* (256x256|1920x1080)"
done
