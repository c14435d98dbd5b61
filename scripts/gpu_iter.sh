set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c2.json 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2>&1
timeout 600 python bench.py --config C3 --driver --steps 3 --warmup 1 > gpurun_out/c3_driver.json 2>&1
timeout 300 python bench.py --config C2 --driver --steps 5 --warmup 2 > gpurun_out/c2_driver.json 2>&1
