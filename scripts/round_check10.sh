timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gpu_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:householder -s 2 -c 1 -o gpurun_out/src_c3_qr python bench.py --config C3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c3_qr.log 2>&1
