#!/bin/bash
# how the two queues of a wavefront share the SMs: filter grid (CTAs per SM), exact grid cap, launch order
run() { echo "== $*"; env "$@" python scripts/frame_breakdown.py 2>&1 | tail -1 | cut -c1-135; }
run A=1
run KNF_EXACT_FIRST=1
run KNF_FILTER_GRID=5
run KNF_FILTER_GRID=4
run KNF_FILTER_GRID=3
run KNF_FILTER_GRID=4 KNF_EXACT_GRID=6
run KNF_FILTER_GRID=4 KNF_EXACT_GRID=6 KNF_EXACT_FIRST=1
run KNF_FILTER_GRID=3 KNF_EXACT_GRID=8 KNF_EXACT_FIRST=1
run KNF_FILTER_GRID=5 KNF_EXACT_GRID=3 KNF_EXACT_FIRST=1
run KNF_EXACT_GRID=4 KNF_EXACT_FIRST=1
run KNF_EXACT_GRID=2 KNF_EXACT_FIRST=1
