# round-1 profiling of the C2 step: tests, bench, launch list, ncu --set full of the top kernels
python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gpu_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for k in householder_qr stage_kernel evaldiff_jobs invert_tiles; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_c2_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
