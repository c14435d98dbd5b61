set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "complex or batched or exponent or library or ledger or residual_sampling or owner_beta" > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
timeout 300 python scripts/trace_batch.py 2 > gpurun_out/trace_batch_k2.json 2>&1
timeout 300 python scripts/trace_batch.py 4 > gpurun_out/trace_batch_k4.json 2>&1
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2>&1
