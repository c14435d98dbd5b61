timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gpu_tests.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>&1
timeout 900 python bench.py --config C4 --steps 2 --warmup 2 > gpurun_out/bench_c4.json 2>&1
timeout 900 python bench.py --config C4 --steps 3 --warmup 2 --reuse-qr > gpurun_out/bench_c4_reuse.json 2>&1
python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2>&1
bash scripts/launches.sh
