set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -v -p no:cacheprovider --timeout 300 > gpurun_out/t5.log 2>&1; echo "rc=$?" >> gpurun_out/t5.log
timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2c.json 2>&1
