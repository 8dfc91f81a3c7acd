#!/bin/bash
# Results table (all configs x tree / merged / collapse) + one full ncu capture of the c5 leaf kernel
tag=${1:-r01m}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 3
timeout 600 python tools/quick.py 1,2,3,4,5 > gpurun_out/${tag}_quick_tree.log 2>&1
QUICK_MERGE=1 timeout 600 python tools/quick.py 1,2,3,4,5 > gpurun_out/${tag}_quick_merged.log 2>&1
QUICK_METHOD=1 timeout 600 python tools/quick.py 1,2,3,4,5 > gpurun_out/${tag}_quick_collapse.log 2>&1
timeout 300 python tools/prof_step.py 5 1 > gpurun_out/${tag}_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:k_leaf2 -c 1 -o gpurun_out/${tag}_c5_leaf2 python tools/prof_step.py 5 1 > gpurun_out/${tag}_ncu.log 2>&1
ls -la gpurun_out
