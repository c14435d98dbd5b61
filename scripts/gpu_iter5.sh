set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2>&1
NS_QR_THREADS=256 timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3_qr256.json 2>&1
NS_QR_THREADS=256 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k C3 > gpurun_out/gpu_tests_qr256.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_qr256.log
