#!/bin/bash
# A/B of occupancy variants + ncu capture of the default c5 leaf kernel
tag=${1:-r01r}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 3
bash tools/ab.sh 4,5 _ab/lib_LEAF2_MINB_CPLX_3.so _ab/lib_LEAF2_MINB_CPLX_3__DLEAF2_ROWS_CPLX_2.so _ab/lib_LEAF2_MINB_4.so > gpurun_out/${tag}_ab.log 2>&1
timeout 300 python tools/prof_step.py 5 1 > gpurun_out/${tag}_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:k_leaf -c 2 -o gpurun_out/${tag}_c5_leaf python tools/prof_step.py 5 1 > gpurun_out/${tag}_ncu.log 2>&1
