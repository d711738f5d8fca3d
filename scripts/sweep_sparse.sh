#!/bin/bash
for cfg in "8 2" "16 4" "32 8" "32 16" "64 16" "128 16"; do set -- $cfg; echo "== KNF_SPARSE_INNER=$1 KNF_SPARSE_KEEP=$2"; KNF_SPARSE_INNER=$1 KNF_SPARSE_KEEP=$2 python scripts/filter_check.py 2>&1 | grep "1080p filter auto\|auto == off"; done
