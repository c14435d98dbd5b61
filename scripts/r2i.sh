set -x
mkdir -p gpurun_out
timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2d.json 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -p no:cacheprovider --timeout 300 -k "batched or complex or exponent" > gpurun_out/t6a.log 2>&1; echo "rc=$?" >> gpurun_out/t6a.log
timeout 3000 python -m pytest tests -m "gpu and slow" -v -p no:cacheprovider --timeout 900 > gpurun_out/t6.log 2>&1; echo "rc=$?" >> gpurun_out/t6.log
