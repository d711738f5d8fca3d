#!/bin/bash
# tail-kernel variants (KNF_TAIL_MIN_BLOCKS = 2 / 3 / 4 / 5 CTAs of 4 warps per SM -> register budget) x hand-over thresholds
for lib in paper_2206_10885_b200/libknf_b200.so paper_2206_10885_b200/libknf_ctail*.so; do
  for t in 24576 49152; do
    echo "== $lib KNF_TAIL=$t"
    KNF_B200_LIB=$PWD/$lib KNF_TAIL=$t KNF_DEBUG_TAIL=1 python scripts/frame_breakdown.py 2>&1 | grep -E "handed over|^frame" | tail -2 | cut -c1-110
  done
done
