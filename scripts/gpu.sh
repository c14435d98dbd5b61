#!/bin/bash
# One documented driver for the GPU box (run it under gpurun from the repo root):
#   gpurun --timeout 3000 -- 'bash scripts/gpu.sh <mode> [args]'
# modes (outputs land in gpurun_out/, merged back by gpurun):
#   tests [pytest -k expr]   pytest -m gpu (+ smoke), log in gpurun_out/tests.log
#   bench [bench args]       bench.py (default: the N=1 headline line) -> gpurun_out/bench.json
#   launches <config>        ncu launch list (gpu__time_duration, cold cache) of 2 steps
#   fp64 <config>            ncu FP64 counters (dadd/dmul/dfma, fp64 pipe, spills, dram) per launch
#   full <config> <regex>    ncu --set full of one launch of the kernel matching regex
#   sanitize <tool>          compute-sanitizer (racecheck|synccheck|memcheck) on a C1/C2-sized run
set -x
mode=$1; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum
case $mode in
  tests)
    timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -s "$@" > gpurun_out/tests.log 2>&1; echo "rc=$?" >> gpurun_out/tests.log
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log ;;
  bench)
    timeout 900 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err ;;
  launches)
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv \
      python scripts/one_step.py $1 2 > gpurun_out/launches_$1.log 2>&1 ;;
  fp64)
    timeout 1200 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/fp64_$1.csv \
      python scripts/one_step.py $1 1 > gpurun_out/fp64_$1.log 2>&1 ;;
  full)
    # the .ncu-rep stays on the box (gpurun_out is capped at 64 MiB): summaries come back
    mkdir -p /tmp/ncu
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o /tmp/ncu/full_$1_$2 \
      python scripts/one_step.py $1 1 > gpurun_out/full_$1_$2.log 2>&1
    python scripts/ncu_summary.py gpurun_out/full_$1_$2.json /tmp/ncu/full_$1_$2.ncu-rep >> gpurun_out/full_$1_$2.log 2>&1
    ncu -i /tmp/ncu/full_$1_$2.ncu-rep --page source --csv 2>/dev/null | python scripts/source_hot.py > gpurun_out/full_$1_$2_hot.txt 2>&1
    ncu -i /tmp/ncu/full_$1_$2.ncu-rep --page source --print-source cuda --csv 2>/dev/null | python scripts/source_hot.py 60 > gpurun_out/full_$1_$2_hot_cuda.txt 2>&1 ;;
  sanitize)
    for C in C1 C2; do
      timeout 600 compute-sanitizer --tool $1 --print-limit 20 python scripts/one_step.py $C 0 > gpurun_out/sanitize_$1_$C.log 2>&1
      echo "rc=$?" >> gpurun_out/sanitize_$1_$C.log
    done
    timeout 600 compute-sanitizer --tool $1 --print-limit 20 python scripts/one_step.py C5 0 2 8 > gpurun_out/sanitize_$1_C5b8.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_$1_C5b8.log ;;
esac
