#!/bin/bash
# Round-2 ncu session: the bench command's launch list (cold, serialised: compare shares) and full
# captures of the dominant launches (config 5 fused + source-task k_leaf2_sym3, config 4 k_leaf2,
# config 5 unfused k_front).  Each ncu command runs only after the same command exited 0 without ncu.
tag=${1:-r02E}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 3
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $B > gpurun_out/${tag}_bench_plain.json 2> gpurun_out/${tag}_bench_plain.err && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${tag}_launches_bench.csv $B > /dev/null 2> gpurun_out/${tag}_ncu_bench.err
timeout 300 python tools/prof_step.py 5 1 > gpurun_out/${tag}_p5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf2_sym3 -c 2 \
    -o gpurun_out/${tag}_c5_leaf2 python tools/prof_step.py 5 1 > /dev/null 2>&1
timeout 300 python tools/prof_step.py 4 1 > gpurun_out/${tag}_p4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf2 -c 1 \
    -o gpurun_out/${tag}_c4_leaf2 python tools/prof_step.py 4 1 > /dev/null 2>&1
ls -la gpurun_out | grep $tag
