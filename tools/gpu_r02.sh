#!/bin/bash
# One GPU-box session of round 2 (at most ONE ncu or compute-sanitizer tool per gpurun call).
# usage: bash tools/gpu_r02.sh <tag> <step>...
#   plain   : build, pytest -m gpu, smoke, bench (driver K/W), plain runs of the ncu/sanitizer commands
#   test | smoke | bench | plainruns : the pieces of `plain`
#   ctr     : ncu FP64 counters of the dominant leaf launch (c3, c4, c5 tree; c5 merged) + launch lists
#   memcheck | racecheck | synccheck | initcheck : compute-sanitizer on tools/sanitize_cases.py
tag=${1:-r02}; shift
steps=${@:-plain}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { tail -20 gpurun_out/${tag}_build.log; exit 3; }
NCU_M=sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum
ctr_runs() {   # plain run && the same command under ncu (FP64 counters of the dominant launch)
  for cv in "3 tree" "4 tree" "5 tree" "5 merged"; do
    set -- $cv
    timeout 300 python tools/fp64_counters.py --run --config $1 --variant $2 > gpurun_out/${tag}_plainctr_c$1_$2.json 2>&1 && \
    timeout 900 ncu --metrics $NCU_M --clock-control none --csv --log-file gpurun_out/ctr_c$1_$2.csv \
      python tools/fp64_counters.py --run --config $1 --variant $2 > gpurun_out/ctr_c$1_$2.json 2> gpurun_out/ctr_c$1_$2.err
  done
}
for s in $steps; do
  case $s in
    plain) bash $0 $tag test smoke bench plainruns ;;
    full) bash $0 $tag test smoke bench nccl checked shards ;;
    test)  timeout 1800 python -m pytest tests -m gpu -q -x -rA 2>&1 | tail -60 > gpurun_out/${tag}_pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1 ;;
    bench) timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err ;;
    plainruns)
      timeout 600 python tools/sanitize_cases.py > gpurun_out/${tag}_sanitize_plain.log 2>&1 || echo "sanitize plain failed"
      timeout 300 python tools/prof_step.py 5 2 > gpurun_out/${tag}_plain5.log 2>&1
      timeout 300 python tools/prof_step.py 4 2 > gpurun_out/${tag}_plain4.log 2>&1 ;;
    ctr)
      ctr_runs
      timeout 300 python tools/prof_step.py 5 2 > gpurun_out/${tag}_plain5.log 2>&1 && \
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/${tag}_launches_c5.csv python tools/prof_step.py 5 2 > /dev/null 2>&1
      timeout 300 python tools/prof_step.py 4 2 > gpurun_out/${tag}_plain4.log 2>&1 && \
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/${tag}_launches_c4.csv python tools/prof_step.py 4 2 > /dev/null 2>&1 ;;
    shards) for c in 4 5; do SHARD_PHASES=1 timeout 900 python tools/shard_times.py $c 2 4 8 > gpurun_out/${tag}_shards_c$c.txt 2>&1; done ;;
    pyt) timeout 1800 python -m pytest $PYT -q -x --tb=long 2>&1 | tail -150 > gpurun_out/${tag}_pyt.log ;;
    nccl) NCCL_DEBUG=INFO timeout 900 python -m pytest tests/test_gpu_nccl.py -q -s 2>&1 | grep -E "NCCL INFO|passed|failed|Error" | head -80 > gpurun_out/${tag}_nccl.log ;;
    checked) timeout 1500 python tools/checked_run.py > gpurun_out/${tag}_checked_run.txt 2>&1 ;;
    memcheck|racecheck|synccheck|initcheck)
      timeout 2400 compute-sanitizer --tool $s --error-exitcode 9 --print-limit 50 \
        python tools/sanitize_cases.py > gpurun_out/${tag}_san_$s.log 2>&1
      echo "exit $?" >> gpurun_out/${tag}_san_$s.log ;;
  esac
done
ls gpurun_out | tail -40
