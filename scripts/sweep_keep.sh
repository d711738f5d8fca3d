#!/bin/bash
for cfg in "12 2" "12 3" "16 3" "16 4" "24 4" "12 1"; do set -- $cfg; echo "== KNF_FILTER_INNER=$1 KNF_FILTER_KEEP=$2"; KNF_FILTER_INNER=$1 KNF_FILTER_KEEP=$2 python scripts/frame_breakdown.py 2>&1 | grep "^frame" | cut -c1-200; done
