#!/bin/bash
for d in 4 8 16 32; do echo "== KNF_SPARSE_DIV=$d"; KNF_SPARSE_DIV=$d python scripts/filter_check.py 2>&1 | grep "1080p filter auto"; done
