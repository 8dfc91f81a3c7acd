#!/bin/bash
# One GPU-box session: tests, smoke, bench, ncu launch list + full captures of the leaf kernels
# (config 5: pass 2's source-task launch and pass 3's fused launch of k_leaf2_sym3; config 4: k_leaf2).
# usage: bash tools/gpu_round.sh <tag> [what...]   what in {test,smoke,bench,ncu,ncufull}
tag=${1:-r01}; shift
what=${@:-test smoke bench ncu ncufull}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_gpu.txt
python -c "import __graft_entry__ as g; g.build()" || exit 3
for w in $what; do
  case $w in
    test)  timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/${tag}_pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1 ;;
    bench) timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err ;;
    ncu)   timeout 300 python tools/prof_step.py 5 2 > gpurun_out/${tag}_plain.log 2>&1 && \
           timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
             --log-file gpurun_out/${tag}_launches_c5.csv python tools/prof_step.py 5 2 > gpurun_out/${tag}_ncu1.log 2>&1 ;
           timeout 300 python tools/prof_step.py 4 2 > gpurun_out/${tag}_plain4.log 2>&1 && \
           timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
             --log-file gpurun_out/${tag}_launches_c4.csv python tools/prof_step.py 4 2 > gpurun_out/${tag}_ncu2.log 2>&1 ;;
    ncufull) timeout 300 python tools/prof_step.py 5 1 > gpurun_out/${tag}_plain5.log 2>&1 && \
           timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
             -k regex:k_leaf2 -c 2 -o gpurun_out/${tag}_c5_leaf2 python tools/prof_step.py 5 1 > gpurun_out/${tag}_ncu3.log 2>&1 ;
           timeout 300 python tools/prof_step.py 4 1 > gpurun_out/${tag}_plain4b.log 2>&1 && \
           timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
             -k regex:k_leaf2 -c 1 -o gpurun_out/${tag}_c4_leaf2 python tools/prof_step.py 4 1 > gpurun_out/${tag}_ncu4.log 2>&1 ;;
  esac
done
ls -la gpurun_out
