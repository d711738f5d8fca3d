#!/bin/bash
# tile-residency cap sweep (KNF_MARCH_MAX_INNER): 1080p random-init frame time, exact mode + decision filter
for k in 4 8 12 16 24 32 64; do
  echo "== KNF_MARCH_MAX_INNER=$k"
  KNF_MARCH_MAX_INNER=$k python scripts/quick_time.py fp32_chain 2>&1 | grep 1080p
done
