set -x
M=gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum
for C in C2 C3; do
timeout 900 ncu --metrics $M --clock-control none -s 30 -c 12 --csv --log-file gpurun_out/r2_fp64_$C.csv python bench.py --config $C --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_fp64_$C.log 2>&1
done
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c3_base.json 2>&1
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c5_base.json 2>&1
nproc > gpurun_out/r2_nproc.txt; python -c "import os; print(len(os.sched_getaffinity(0)))" >> gpurun_out/r2_nproc.txt; lscpu | head -20 >> gpurun_out/r2_nproc.txt
