set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_staggered.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for t in 64 128 256; do
NS_STAGE2_THREADS=$t timeout 120 python scripts/trace_stage.py C2 > gpurun_out/tst_c2_$t.json 2>&1
NS_STAGE2_THREADS=$t timeout 300 python scripts/trace_stage.py C3 > gpurun_out/tst_c3_$t.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c2.json 2>&1
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3.json 2>&1
