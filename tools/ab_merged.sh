#!/bin/bash
# A/B timing of library variants on the midpoint-merged path: bash tools/ab_merged.sh "4,5" lib1.so ...
cfg=$1; shift
echo "== default"; QUICK_MERGE=1 python tools/quick.py $cfg 2>&1 | grep -E "^c[0-9]" | cut -c1-110
for l in "$@"; do echo "== $l"; SG_B200_LIB=$PWD/$l QUICK_MERGE=1 python tools/quick.py $cfg 2>&1 | grep -E "^c[0-9]" | cut -c1-110; done
