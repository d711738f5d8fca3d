#!/bin/bash
# A/B filter-kernel variants built as paper_2206_10885_b200/libknf_v*.so (KNF_B200_LIB override)
for lib in paper_2206_10885_b200/libknf_b200.so paper_2206_10885_b200/libknf_v*.so; do
  echo "== $lib"
  KNF_B200_LIB=$PWD/$lib python scripts/quick_time.py fp32_chain 2>&1 | grep 1080p
done
