#!/bin/bash
# A/B timing of library variants: bash tools/ab.sh "4,5" lib1.so lib2.so ...
cfg=$1; shift
echo "== default"; python tools/quick.py $cfg 2>&1 | grep -E "^c[0-9]" | cut -c1-110
for l in "$@"; do echo "== $l"; SG_B200_LIB=$PWD/$l python tools/quick.py $cfg 2>&1 | grep -E "^c[0-9]" | cut -c1-110; done
