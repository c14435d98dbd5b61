set -x
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 120 python scripts/trace_stage.py C2 > gpurun_out/tst_c2.json 2>&1
timeout 300 python scripts/trace_stage.py C3 > gpurun_out/tst_c3.json 2>&1
timeout 300 env NS_CQR_TRACE=1 python scripts/trace_qr.py C2 > gpurun_out/tqr_c2.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c2.json 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2>&1
NS_QR_THREADS=256 timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3_qr256.json 2>&1
