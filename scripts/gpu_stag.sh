set -x
timeout 900 python -m pytest tests/test_gpu_staggered.py -m gpu -q -p no:cacheprovider -x > gpurun_out/stag_tests.log 2>&1; echo "rc=$?" >> gpurun_out/stag_tests.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_staggered.py > gpurun_out/gpu_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests2.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c2_after_window.json 2>&1
