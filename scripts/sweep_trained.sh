#!/bin/bash
# residency / sparse-kernel knobs on the trained fields (exact FP32 path only)
run() { echo "== $*"; for f in trained8 trained16; do env "$@" python scripts/frame_breakdown.py $f 2>&1 | tail -1 | cut -c1-110; done; }
run A=1
run KNF_MARCH_MAX_INNER=4
run KNF_MARCH_MAX_INNER=6
run KNF_MARCH_MAX_INNER=12
run KNF_SPARSE_DIV=4
run KNF_SPARSE_DIV=16
run KNF_SPARSE_INNER=4
run KNF_SPARSE_INNER=12
run KNF_TAIL=12288
run KNF_TAIL=36864
