#!/bin/bash
for lib in paper_2206_10885_b200/libknf_b200.so paper_2206_10885_b200/libknf_vc*.so; do
  echo "== $lib"
  KNF_B200_LIB=$PWD/$lib python scripts/frame_breakdown.py distilled 2>&1 | grep "^frame" | cut -c1-90
  KNF_B200_LIB=$PWD/$lib KNF_FILTER=off python scripts/frame_breakdown.py 2>&1 | grep "^frame" | cut -c1-90
done
