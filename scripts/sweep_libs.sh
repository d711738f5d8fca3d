#!/bin/bash
# A/B kernel variants built as paper_2206_10885_b200/libknf_*.so (KNF_B200_LIB override)
for lib in paper_2206_10885_b200/libknf_b200.so paper_2206_10885_b200/libknf_c*.so; do
  echo "== $lib"
  KNF_B200_LIB=$PWD/$lib python scripts/gpu_probe.py 2>&1 | grep -E "sdf_query M=4194304|render .* 1920x1080" | cut -c1-150
done
