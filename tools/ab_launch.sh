#!/bin/bash
# A/B of library variants with the per-launch device times: bash tools/ab_launch.sh "3,5" lib1.so ...
cfg=$1; shift
run() { python tools/quick.py $cfg 2>&1 | grep -E "^c[0-9]|launches" | sed -E 's/(plan=[0-9.]+ms )//' | cut -c1-150; }
echo "== default"; run
for l in "$@"; do echo "== $l"; SG_B200_LIB=$PWD/$l run; done
echo "== default (again)"; run
