#!/bin/bash
# knob sweep after the refined Lipschitz bounds made the filter cheap: which side of a wavefront is the critical path now?
run() { echo "== $*"; env "$@" python scripts/frame_breakdown.py 2>&1 | tail -1 | cut -c1-330; }
run A=1
run KNF_SPARSE_DIV=16
run KNF_SPARSE_DIV=64
run KNF_SPARSE_DIV=100000
run KNF_SPARSE_SMALL=0
run KNF_SPARSE_INNER=16 KNF_SPARSE_KEEP=4
run KNF_SPARSE_INNER=32 KNF_SPARSE_KEEP=8
run KNF_TAIL=49152
run KNF_TAIL=98304
run KNF_TAIL=12288
run KNF_FILTER_INNER=8
run KNF_FILTER_INNER=24
run KNF_FILTER_GRID=4
run KNF_OVERLAP=0
run KNF_MARCH_MAX_INNER=16
