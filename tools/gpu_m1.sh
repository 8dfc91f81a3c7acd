set -x
python -c "import __graft_entry__ as g; g.build()" || exit 3
timeout 900 python bench.py > gpurun_out/r01i_bench.json 2> gpurun_out/r01i_bench.err
QUICK_MERGE=1 timeout 300 python tools/prof_step.py 5 1 > gpurun_out/r01i_m5_plain.log 2>&1 && \
QUICK_MERGE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01i_launches_m5.csv python tools/prof_step.py 5 2 > gpurun_out/r01i_ncu1.log 2>&1
QUICK_MERGE=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_leaf2 -c 1 -o gpurun_out/r01i_m5_leaf2 python tools/prof_step.py 5 1 > gpurun_out/r01i_ncu2.log 2>&1
QUICK_MERGE=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_leaf2 -c 1 -o gpurun_out/r01i_m4_leaf2 python tools/prof_step.py 4 1 > gpurun_out/r01i_ncu3.log 2>&1
ls gpurun_out | grep r01i
